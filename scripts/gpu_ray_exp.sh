# Ray-kernel experiment builds (RAY_EXP variants, on the box): stage times of one cfg3 frame.
mkdir -p /tmp/rx
OBJS=$(ls build/obj/*.o | grep -v raymarch.o)
for e in ${EXPS:-1 2 6}; do
  (nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Iinclude \
    -Ipaper_2409_10876_b200/csrc --expt-relaxed-constexpr -DRAY_EXP=$e \
    -c paper_2409_10876_b200/csrc/raymarch.cu -o /tmp/rx/r$e.o &&
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/rx/lib$e.so $OBJS /tmp/rx/r$e.o -lcudart) &
done
wait
echo "base $(python scripts/profile_iter.py --steps 1 2>&1 | tail -1 | grep -o "ray_backward.: [0-9.]*")"
for e in ${EXPS:-1 2 6}; do echo "exp$e $(PACT_LIB=/tmp/rx/lib$e.so python scripts/profile_iter.py --steps 1 2>&1 | tail -1 | grep -o "ray_backward.: [0-9.]*")"; done

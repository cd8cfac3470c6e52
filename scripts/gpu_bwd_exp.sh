# Timing experiments of the fused SIREN backward (BWD_EXP variants built on the box).
mkdir -p /tmp/bx gpurun_out
OBJS=$(ls build/obj/*.o | grep -v siren_bwd.o)
for e in ${EXPS:-1 2 3 4}; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Iinclude \
    -Ipaper_2409_10876_b200/csrc --expt-relaxed-constexpr -DBWD_EXP=$e $EXTRA \
    -c paper_2409_10876_b200/csrc/siren_bwd.cu -o /tmp/bx/b$e.o &&
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/bx/lib$e.so $OBJS /tmp/bx/b$e.o -lcudart &
done
wait
echo exp0; python scripts/profile_iter.py --steps 1 2>&1 | tail -1
for e in ${EXPS:-1 2 3 4}; do echo exp$e; PACT_LIB=/tmp/bx/lib$e.so python scripts/profile_iter.py --steps 1 2>&1 | tail -1; done

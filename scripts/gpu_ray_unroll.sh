# Ray-kernel unroll variants (built on the box): cfg3 stage times and cfg5 stage times.
mkdir -p /tmp/ru
OBJS=$(ls build/obj/*.o | grep -v raymarch.o)
V="${V:-4_4 8_4 4_8 8_8}"
for v in $V; do
  IFS=_ read f b <<< "$v"
  (nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Iinclude \
    -Ipaper_2409_10876_b200/csrc --expt-relaxed-constexpr -DRAY_FWD_UNROLL=$f -DRAY_BWD_BATCH=$b \
    -c paper_2409_10876_b200/csrc/raymarch.cu -o /tmp/ru/r$v.o &&
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/ru/lib$v.so $OBJS /tmp/ru/r$v.o -lcudart) &
done
wait
for v in $V; do echo "v$v cfg3 $(PACT_LIB=/tmp/ru/lib$v.so python scripts/profile_iter.py --steps 1 2>&1 | tail -1 | grep -o "wavefront.: [0-9.]*\|ray_backward.: [0-9.]*" | tr '\n' ' ')"; done
for v in ${V5:-4_4 8_8}; do echo "v$v cfg5 $(PACT_LIB=/tmp/ru/lib$v.so timeout 300 python scripts/cfg5_probe.py 2>&1 | grep stages | grep -o "wavefront.: [0-9.]*\|ray_backward.: [0-9.]*" | tr '\n' ' ')"; done

# Buffer-depth variants of the fused SIREN backward (built on the box).
mkdir -p /tmp/bv
OBJS=$(ls build/obj/*.o | grep -v siren_bwd.o)
V="${V:-3_2_3 3_2_2 3_1_4 2_2_4}"
for v in $V; do
  IFS=_ read d z r <<< "$v"
  (nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Iinclude \
    -Ipaper_2409_10876_b200/csrc --expt-relaxed-constexpr -DBWD_ND=$d -DBWD_NZ=$z -DBWD_NR=$r \
    -c paper_2409_10876_b200/csrc/siren_bwd.cu -o /tmp/bv/b$v.o &&
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/bv/lib$v.so $OBJS /tmp/bv/b$v.o -lcudart) &
done
wait
for v in $V; do echo "v$v $(PACT_LIB=/tmp/bv/lib$v.so python scripts/profile_iter.py --steps 1 2>&1 | tail -1 | grep -o "siren_bwd.: [0-9.]*")"; done

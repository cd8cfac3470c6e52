# Forward-chain experiment builds (CHAIN_EXP variants, on the box).
mkdir -p /tmp/cx
OBJS=$(ls build/obj/*.o | grep -v siren_chain.o)
for e in ${EXPS:-1 3}; do
  (nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Iinclude \
    -Ipaper_2409_10876_b200/csrc --expt-relaxed-constexpr -DCHAIN_EXP=$e \
    -c paper_2409_10876_b200/csrc/siren_chain.cu -o /tmp/cx/c$e.o &&
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/cx/lib$e.so $OBJS /tmp/cx/c$e.o -lcudart) &
done
wait
echo "base $(python scripts/profile_iter.py --steps 1 2>&1 | tail -1 | grep -o "siren_fwd.: [0-9.]*")"
for e in ${EXPS:-1 3}; do echo "exp$e $(PACT_LIB=/tmp/cx/lib$e.so python scripts/profile_iter.py --steps 1 2>&1 | tail -1 | grep -o "siren_fwd.: [0-9.]*")"; done

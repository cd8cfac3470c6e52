# Timeline of CTA 0 of the fused SIREN forward (CHAIN_EXP=2 build on the box).
mkdir -p /tmp/cx
OBJS=$(ls build/obj/*.o | grep -v siren_chain.o)
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Iinclude \
  -Ipaper_2409_10876_b200/csrc --expt-relaxed-constexpr -DCHAIN_EXP=2 \
  -c paper_2409_10876_b200/csrc/siren_chain.cu -o /tmp/cx/c2.o &&
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/cx/lib_c2.so $OBJS /tmp/cx/c2.o -lcudart
PACT_LIB=/tmp/cx/lib_c2.so python scripts/chain_trace.py 2>&1 | head -90

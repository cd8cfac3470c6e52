mkdir -p /tmp/bx
OBJS=$(ls build/obj/*.o | grep -v siren_bwd.o)
for m in ${MODES:-1 2}; do
 (nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Iinclude -Ipaper_2409_10876_b200/csrc --expt-relaxed-constexpr -DBWD_EXP=5 -DBWD_TRACE_MODE=$m -c paper_2409_10876_b200/csrc/siren_bwd.cu -o /tmp/bx/t$m.o && nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/bx/libt$m.so $OBJS /tmp/bx/t$m.o -lcudart) &
done
wait
for m in ${MODES:-1 2}; do echo MODE $m; PACT_LIB=/tmp/bx/libt$m.so python scripts/bwd_trace.py 2>&1 | tail -15; done

# Width-256 layer experiments (WIDE_EXP builds on the box): cfg5 SIREN stage times.
mkdir -p /tmp/wx
OBJS=$(ls build/obj/*.o | grep -v siren_wide.o)
for e in ${EXPS:-1}; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Iinclude \
    -Ipaper_2409_10876_b200/csrc --expt-relaxed-constexpr -DWIDE_EXP=$e \
    -c paper_2409_10876_b200/csrc/siren_wide.cu -o /tmp/wx/w$e.o &&
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/wx/lib$e.so $OBJS /tmp/wx/w$e.o -lcudart
done
echo "base $(timeout 500 python scripts/cfg5_probe.py 2>&1 | grep stages)"
for e in ${EXPS:-1}; do echo "exp$e $(PACT_LIB=/tmp/wx/lib$e.so timeout 500 python scripts/cfg5_probe.py 2>&1 | grep stages)"; done

# Build experiment variants of the library (TC_EXP=1..3) into build/exp/.
set -e
mkdir -p build/exp
OBJS=$(ls build/obj/*.o | grep -v siren_tc.o)
for e in 6; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
    -Xcompiler -fPIC -Iinclude -Ipaper_2409_10876_b200/csrc --expt-relaxed-constexpr -DTC_EXP=$e \
    -c paper_2409_10876_b200/csrc/siren_tc.cu -o build/exp/siren_tc_$e.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/exp/libpact_exp$e.so \
    $OBJS build/exp/siren_tc_$e.o -lcudart
done

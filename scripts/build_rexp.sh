set -e
mkdir -p build/exp
OBJS=$(ls build/obj/*.o | grep -v raymarch.o)
for e in 1 5 6; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
    -Xcompiler -fPIC -Iinclude -Ipaper_2409_10876_b200/csrc --expt-relaxed-constexpr -DRAY_EXP=$e \
    -c paper_2409_10876_b200/csrc/raymarch.cu -o build/exp/raymarch_$e.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/exp/libpact_rexp$e.so \
    $OBJS build/exp/raymarch_$e.o -lcudart
done

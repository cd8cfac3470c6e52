set -e
mkdir -p build/exp
OBJS=$(ls build/obj/*.o | grep -v raymarch.o)
for b in 768 800; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
    -Xcompiler -fPIC -Iinclude -Ipaper_2409_10876_b200/csrc --expt-relaxed-constexpr -DRAY_BLOCK=$b \
    -c paper_2409_10876_b200/csrc/raymarch.cu -o build/exp/raymarch_b$b.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/exp/libpact_b$b.so \
    $OBJS build/exp/raymarch_b$b.o -lcudart
done

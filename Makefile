# Builds the sm_100a library, the oracle (CPU restatement) and, when the
# reference tree is mounted, oracle/_ref (the reference compiled as-is).
#   make            -> lib + oracle (+ _ref if /root/reference exists)
#   make lib        -> paper_2409_10876_b200/lib/libpact_cuda.so
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
CC ?= gcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -Wall \
           -Iinclude -Ipaper_2409_10876_b200/csrc --expt-relaxed-constexpr
PKG := paper_2409_10876_b200
LIBDIR := $(PKG)/lib
CU_SRCS := $(wildcard $(PKG)/csrc/*.cu)
CU_OBJS := $(patsubst $(PKG)/csrc/%.cu,build/obj/%.o,$(CU_SRCS))
CU_HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/pact_cuda.h

.PHONY: all lib oracle ref clean

all: lib oracle ref

lib: $(LIBDIR)/libpact_cuda.so

build/obj/%.o: $(PKG)/csrc/%.cu $(CU_HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIBDIR)/libpact_cuda.so: $(CU_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -lcudart

oracle:
	$(MAKE) -C oracle oracle

ref:
	@if [ -d /root/reference/proj/include/pact ]; then $(MAKE) -C oracle ref; \
	 else echo "reference tree absent: keeping prebuilt oracle/_ref"; fi

clean:
	rm -rf build $(LIBDIR)
	$(MAKE) -C oracle clean

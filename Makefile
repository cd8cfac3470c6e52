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

.PHONY: all lib oracle ref pactrec clean

all: lib oracle ref pactrec

lib: $(LIBDIR)/libpact_cuda.so

build/obj/%.o: $(PKG)/csrc/%.cu $(CU_HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIBDIR)/libpact_cuda.so: $(CU_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -lcudart

# pactrec: the reference's CLI driver over the drop-in headers (host C++)
PACTREC := $(PKG)/bin/pactrec
pactrec: $(PACTREC)

$(PACTREC): $(PKG)/tools/pactrec.cpp $(PKG)/tools/cli_args.hpp $(PKG)/tools/json_lite.hpp \
            $(wildcard $(PKG)/include/pact/*.hpp) include/pact_cuda.h $(LIBDIR)/libpact_cuda.so
	@mkdir -p $(PKG)/bin
	$(CXX) -std=c++17 -O2 -Wall -Wextra -pthread -Iinclude -I$(PKG)/include -I$(PKG)/tools -o $@ \
	  $(PKG)/tools/pactrec.cpp -L$(LIBDIR) -lpact_cuda -Wl,-rpath,'$$ORIGIN/../lib'

oracle:
	$(MAKE) -C oracle oracle

ref:
	@if [ -d /root/reference/proj/include/pact ]; then $(MAKE) -C oracle ref; \
	 else echo "reference tree absent: keeping prebuilt oracle/_ref"; fi

clean:
	rm -rf build $(LIBDIR)
	$(MAKE) -C oracle clean

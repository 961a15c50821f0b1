# Build of the B200-native QC hot path.
#   libgqc.so       C-ABI + sm_100a kernels (include/gqc.h)
#   oracle          CPU restatement used only by tests/bench (oracle/)
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       ?= g++
PKG       := paper_2305_14641_b200
CSRC      := $(PKG)/csrc
ARCH      := -gencode arch=compute_100a,code=sm_100a
# -fmad=false: no FMA contraction anywhere (every fp64 add/mul rounds like the
# reference's SSE2 build); host code: no -march, no contraction.
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -Xptxas -v \
             -Xcompiler -fPIC,-O2,-ffp-contract=off,-Wall -I include -I $(CSRC)
LIBGQC    := $(PKG)/libgqc.so
GQC_SRCS  := $(CSRC)/capi.cu $(CSRC)/kernels.cu $(CSRC)/khop.cu $(CSRC)/csr_build.cu $(CSRC)/host_exp.cpp
GQC_HDRS  := include/gqc.h $(CSRC)/gqc_internal.h $(CSRC)/ff_chain.cuh

all: $(LIBGQC) oracle facade

$(LIBGQC): $(GQC_SRCS) $(GQC_HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(GQC_SRCS) 2> $(PKG)/build_ptxas.log || (cat $(PKG)/build_ptxas.log; exit 1)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(LIBGQC) $(PKG)/build_ptxas.log $(LIBFACADE) $(CLI)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean

# graphqc-compatible C++ host facade (reference API) + CLI, on top of libgqc.
HOST      := $(PKG)/host
LIBFACADE := $(PKG)/libgraphqc.so
CLI       := $(PKG)/bin/graphqc
HOSTFLAGS := -O2 -std=c++20 -ffp-contract=off -fPIC -Wall -Wextra -I $(HOST)/include -I include
HOST_SRCS := $(wildcard $(HOST)/src/*.cpp)
HOST_HDRS := $(wildcard $(HOST)/include/graphqc/*.hpp) $(HOST)/src/device.hpp include/gqc.h

facade: $(LIBFACADE) $(CLI)

$(LIBFACADE): $(HOST_SRCS) $(HOST_HDRS) $(LIBGQC)
	$(CXX) $(HOSTFLAGS) -shared -o $@ $(HOST_SRCS) -L$(PKG) -lgqc -Wl,-rpath,'$$ORIGIN'

$(CLI): $(HOST)/tools/graphqc_main.cpp $(LIBFACADE)
	@mkdir -p $(PKG)/bin
	$(CXX) $(HOSTFLAGS) -o $@ $< -L$(PKG) -lgraphqc -lgqc -Wl,-rpath,'$$ORIGIN/..'

.PHONY: facade

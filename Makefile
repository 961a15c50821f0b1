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
GQC_SRCS  := $(CSRC)/capi.cu $(CSRC)/kernels.cu $(CSRC)/host_exp.cpp
GQC_HDRS  := include/gqc.h $(CSRC)/gqc_internal.h

all: $(LIBGQC) oracle

$(LIBGQC): $(GQC_SRCS) $(GQC_HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(GQC_SRCS) 2> $(PKG)/build_ptxas.log || (cat $(PKG)/build_ptxas.log; exit 1)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(LIBGQC) $(PKG)/build_ptxas.log
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean

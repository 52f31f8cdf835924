# Build recipe for the B200 path (sm_100a only) and the CPU checkers.
#   make            -> CUDA layer + host runtime + CPU oracle (+ reference build when present)
#   make cuda host  -> individual pieces
NVCC    ?= nvcc
# the system toolchain (an /opt/gcc wrapper on PATH/CXX produced miscompiled -O2 objects here)
CXX     := $(firstword $(wildcard /usr/bin/g++) g++)
CC      ?= gcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
PKG     := paper_2410_03065_b200
LIB     := $(PKG)/_lib
INC     := -Iinclude
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden -Xptxas -v $(INC)
# experiment-only attention kernels (two-tile, decoupled groups): make ATTN_VARIANTS=1
ifeq ($(ATTN_VARIANTS),1)
NVFLAGS += -DCAKE_ATTN_VARIANTS
endif
CXXFLAGS:= -O3 -std=c++20 -fPIC -Wall -Wextra -Wno-unused-parameter $(INC) -I/usr/local/cuda/include
CUDA_LIBDIR := /usr/local/cuda/lib64

CUDA_SRC := $(PKG)/csrc/cuda/cake_cuda.cu
CUDA_HDR := $(wildcard $(PKG)/csrc/cuda/*.cuh) include/cake_cuda.h
HOST_SRC := $(wildcard $(PKG)/csrc/host/*.cpp)
HOST_HDR := $(wildcard include/cake/*.hpp) include/cake_c.h include/cake_cuda.h

all: cuda host oracle

cuda: $(LIB)/libcake_cuda.so
host: $(LIB)/libcake.so

$(LIB)/libcake_cuda.so: $(CUDA_SRC) $(CUDA_HDR)
	@mkdir -p $(LIB)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(CUDA_SRC) -L$(CUDA_LIBDIR) -lnccl 2> $(LIB)/ptxas_cuda.log || (cat $(LIB)/ptxas_cuda.log; false)

$(LIB)/libcake.so: $(HOST_SRC) $(HOST_HDR) $(LIB)/libcake_cuda.so
	$(CXX) $(CXXFLAGS) -shared -o $@ $(HOST_SRC) -L$(LIB) -lcake_cuda -Wl,-rpath,'$$ORIGIN' \
	    -L$(CUDA_LIBDIR) -lcudart -lcrypto -lpthread -Wl,-Bsymbolic

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all cuda host oracle clean

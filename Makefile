# Build everything in-tree (the .so files travel to the GPU box with gpurun).
#   make            -> synth, oracle, CUDA library
#   make synth | oracle | lib
CC      := gcc
CXX     := g++
NVCC    ?= /usr/local/cuda/bin/nvcc
CUDA    ?= /usr/local/cuda

PKG     := paper_1704_02083_b200
CSRC    := $(PKG)/csrc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Xptxas -v \
           --expt-relaxed-constexpr
CUDA_SRCS := $(wildcard $(CSRC)/*.cu)
CPP_SRCS  := $(wildcard $(CSRC)/*.cpp)
CSRC_HDRS := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/rapid.h

all: synth oracle lib

synth: synth/libsynth.so
synth/libsynth.so: synth/synth.c
	$(CC) -O2 -fopenmp -fPIC -shared -o $@ $<

# The oracle is plain, single-threaded C (no OpenMP, no vectorisation pragmas).
oracle: oracle/liboracle.so
oracle/liboracle.so: oracle/oracle.c oracle/oracle.h
	$(CC) -O2 -std=gnu11 -fPIC -shared -Wall -Wextra -o $@ oracle/oracle.c

lib: $(PKG)/librapid.so
$(PKG)/librapid.so: $(CUDA_SRCS) $(CPP_SRCS) $(CSRC_HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(CUDA_SRCS) $(CPP_SRCS) -lcuda 2> build_ptxas.log || (cat build_ptxas.log; exit 1)

clean:
	rm -f synth/libsynth.so oracle/liboracle.so $(PKG)/librapid.so build_ptxas.log

.PHONY: all synth oracle lib clean

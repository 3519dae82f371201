# Build the sm_100a engine in-tree (the .so travels to the GPU box with gpurun).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -fmad=false -Xcompiler -fPIC,-ffp-contract=off -shared -lnccl
SRC := paper_2510_10891_b200/csrc/hpr_engine.cu paper_2510_10891_b200/csrc/hpr_screen.cu paper_2510_10891_b200/csrc/hpr_presolve.cpp
DEPS := $(SRC) $(wildcard paper_2510_10891_b200/csrc/*.cuh) $(wildcard paper_2510_10891_b200/csrc/*.h) include/hprlp_b200.h include/hpr_presolve.h include/hpr_screen.h
LIB := paper_2510_10891_b200/libhprlp_b200.so

all: $(LIB)

$(LIB): $(DEPS)
	$(NVCC) $(FLAGS) -o $@ $(SRC)

clean:
	rm -f $(LIB)

.PHONY: all clean

# Builds the sm_100a C-ABI library in-tree (it travels to the GPU box with gpurun).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v -diag-suppress 20208 --expt-relaxed-constexpr
SRC := $(wildcard paper_2009_05473_b200/csrc/*.cu)
HDR := $(wildcard paper_2009_05473_b200/csrc/*.cuh) include/sfw3d_cuda.h
LIB := paper_2009_05473_b200/_lib/libsfw3d_cuda.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) -lcudart -lpthread 2> build_ptxas.log || (cat build_ptxas.log; exit 1)

oracle:
	$(MAKE) -C oracle

clean:
	rm -f $(LIB) build_ptxas.log

.PHONY: all clean oracle

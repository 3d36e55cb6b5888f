# Builds the sm_100a C-ABI library in-tree (it travels to the GPU box with gpurun).
# One object per translation unit (parallel with -j); no relocatable device
# code is needed: device helpers are header-inline, cross-file calls are host.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fopenmp -Xptxas -v -diag-suppress 20208 --expt-relaxed-constexpr
SRC := $(wildcard paper_2009_05473_b200/csrc/*.cu)
HDR := $(wildcard paper_2009_05473_b200/csrc/*.cuh) include/sfw3d_cuda.h
OBJDIR := build/obj
OBJ := $(patsubst paper_2009_05473_b200/csrc/%.cu,$(OBJDIR)/%.o,$(SRC))
LIB := paper_2009_05473_b200/_lib/libsfw3d_cuda.so

all: $(LIB)

$(OBJDIR)/%.o: paper_2009_05473_b200/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(LIB): $(OBJ)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart -lcufft -lgomp -lpthread
	@cat $(OBJDIR)/*.ptxas.log > build_ptxas.log

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(LIB) $(OBJDIR) build_ptxas.log

.PHONY: all clean oracle

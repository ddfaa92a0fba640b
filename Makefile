# Two independent build products that share no sources:
#   oracle  -> oracle/liboracle.so                  (plain C CPU oracle, test infrastructure)
#   lib     -> paper_1904_06376_b200/libbf16x.so    (the product: CUDA kernels + C ABI, sm_100a)
NVCC    ?= /usr/local/cuda/bin/nvcc
PKG     := paper_1904_06376_b200
CSRC    := $(PKG)/csrc
CU_SRCS := $(wildcard $(CSRC)/*.cu)
CU_HDRS := $(wildcard $(CSRC)/*.cuh) include/bf16x.h
GENCODE := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(GENCODE) -lineinfo -Xcompiler -fPIC -Iinclude -I$(CSRC) \
           --expt-relaxed-constexpr -Xptxas -v

.PHONY: all oracle lib clean
all: oracle lib

oracle: oracle/liboracle.so
oracle/liboracle.so: oracle/bf16x_oracle.c
	gcc -O3 -march=x86-64-v3 -fno-fast-math -ffp-contract=off -fopenmp -fPIC -shared -std=gnu99 -o $@ $< -lm

lib: $(PKG)/libbf16x.so
$(PKG)/libbf16x.so: $(CU_SRCS) $(CU_HDRS)
	$(NVCC) $(NVFLAGS) -shared -cudart static -o $@ $(CU_SRCS) 2> build_ptxas.log || (cat build_ptxas.log; false)

clean:
	rm -f oracle/liboracle.so $(PKG)/libbf16x.so

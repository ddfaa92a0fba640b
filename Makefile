# Two independent build products that share no sources:
#   oracle  -> oracle/liboracle.so                  (plain C CPU oracle, test infrastructure)
#   lib     -> paper_1904_06376_b200/libbf16x.so    (the product: CUDA kernels + C ABI, sm_100a)
# The CUDA sources compile to objects in parallel (the K2 kernel is instantiated per variant in
# gemm_v<V>.cu) and link into one shared library with the static CUDA runtime.
NVCC    ?= /usr/local/cuda/bin/nvcc
PKG     := paper_1904_06376_b200
CSRC    := $(PKG)/csrc
OBJDIR  := build/obj
CU_SRCS := $(wildcard $(CSRC)/*.cu)
CU_OBJS := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS))
CU_HDRS := $(wildcard $(CSRC)/*.cuh) include/bf16x.h
GENCODE := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(GENCODE) -lineinfo -Xcompiler -fPIC -Iinclude -I$(CSRC) \
           --expt-relaxed-constexpr -Xptxas -v
MAKEFLAGS += -j8

.PHONY: all oracle lib clean trace variant
all: oracle lib

oracle: oracle/liboracle.so
oracle/liboracle.so: oracle/bf16x_oracle.c
	gcc -O3 -march=x86-64-v3 -fno-fast-math -ffp-contract=off -fopenmp -fPIC -shared -std=gnu99 -o $@ $< -lm

lib: $(PKG)/libbf16x.so
$(OBJDIR)/%.o: $(CSRC)/%.cu $(CU_HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(PKG)/libbf16x.so: $(CU_OBJS)
	$(NVCC) $(GENCODE) -shared -cudart static -o $@ $(CU_OBJS)
	cat $(OBJDIR)/*.ptxas.log > build_ptxas.log

# diagnostic build with the per-CTA %globaltimer trace compiled in (tools/gemm_trace.py loads it
# through BF16X_LIB=build/trace/libbf16x.so); never the product library
TRACE_OBJS := $(patsubst $(CSRC)/%.cu,build/trace/%.o,$(CU_SRCS))
build/trace/%.o: $(CSRC)/%.cu $(CU_HDRS)
	@mkdir -p build/trace
	$(NVCC) $(NVFLAGS) -DBF16X_TRACE -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; false)
trace: build/trace/libbf16x.so
build/trace/libbf16x.so: $(TRACE_OBJS)
	$(NVCC) $(GENCODE) -shared -cudart static -o $@ $(TRACE_OBJS)

# A/B build of the library with extra compile flags (probes only):
#   make variant VDIR=build/epi4 VFLAGS=-DBF16X_EPI_NBUF=4  ->  BF16X_LIB=build/epi4/libbf16x.so
VDIR ?= build/variant
VFLAGS ?=
VAR_OBJS := $(patsubst $(CSRC)/%.cu,$(VDIR)/%.o,$(CU_SRCS))
$(VDIR)/%.o: $(CSRC)/%.cu $(CU_HDRS)
	@mkdir -p $(VDIR)
	$(NVCC) $(NVFLAGS) $(VFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; false)
variant: $(VDIR)/libbf16x.so
$(VDIR)/libbf16x.so: $(VAR_OBJS)
	$(NVCC) $(GENCODE) -shared -cudart static -o $@ $(VAR_OBJS)

clean:
	rm -rf oracle/liboracle.so $(PKG)/libbf16x.so $(OBJDIR)

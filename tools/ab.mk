# developer A/B builds of libhps_b200 with compile-time variants (not part of the product build):
#   mkdir -p build_ab && make -C build_ab -f ../tools/ab.mk VARIANT=pull DEFS=-DHPS_PANEL_PUSH=0
NVCC ?= /usr/local/cuda/bin/nvcc
SRCDIR := ../paper_2503_17535_b200/csrc
SRC := gemm.cu lu.cu hps_kernels.cu leaf_fused.cu leaf_fdm.cu gemv.cu hps_ctx.cu general.cu output.cu sharded.cu geometry.cpp tree_general.cpp
FLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -ccbin /usr/bin/g++ --expt-relaxed-constexpr
# usage: make VARIANT=pull DEFS=-DHPS_PANEL_PUSH=0
VARIANT ?= ab
lib_$(VARIANT).so: $(addprefix $(SRCDIR)/,$(SRC))
	mkdir -p o_$(VARIANT)
	for f in $(SRC); do $(NVCC) $(FLAGS) $(DEFS) -c $(SRCDIR)/$$f -o o_$(VARIANT)/$$f.o || exit 1; done
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -shared -o $@ o_$(VARIANT)/*.o -lcudart -lpthread

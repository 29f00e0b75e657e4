# Builds the HGF C-ABI shared library for B200 (sm_100a).
# The per-channel-count kernels are compiled once per n (hgf_inst.cu with -DHGF_N=n) so make -j
# builds them in parallel.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr
PKG := paper_1803_00005_b200
CS := $(PKG)/csrc
NS := 1 2 3 4 5 6 7 8 9 10 11 12 13 14 15 16 17 18 19 20
DEPS := $(wildcard $(CS)/*.cuh) $(wildcard $(CS)/*.h) include/hgf.h
MDS := 1_1 1_2 1_3 2_1 2_2 2_3 3_1 3_2 3_3 4_1 5_1 6_1 4_2
OBJ := build/hgf_api.o build/hgf_dispatch.o build/hgf_stereo.o build/hgf_coef5.o build/hgf_agg5.o build/hgf_agg6.o build/hgf_agg6w.o $(foreach n,$(NS),build/inst_$(n).o) $(foreach md,$(MDS),build/inst2_$(md).o)
LIB := $(PKG)/libhgf.so

all: $(LIB)

build/hgf_%.o: $(CS)/hgf_%.cu $(DEPS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

build/inst_%.o: $(CS)/hgf_inst.cu $(DEPS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -DHGF_N=$* -c $< -o $@

build/inst2_%.o: $(CS)/hgf_inst2.cu $(DEPS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -DHGF_M=$(word 1,$(subst _, ,$*)) -DHGF_D=$(word 2,$(subst _, ,$*)) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

clean:
	rm -rf build $(LIB)

.PHONY: all clean

# Product build: sm_100a CUDA kernels + C-ABI -> paper_2306_16926_b200/libosp_b200.so
# (in-tree, so it travels to the GPU box with gpurun and is what tests/bench load).
#
#   make            -> library + oracle/liboracle.so
#   make ref        -> oracle/_ref/ (needs /root/reference; test infrastructure)

NVCC ?= nvcc
PKG := paper_2306_16926_b200
CSRC := $(PKG)/csrc
LIB := $(PKG)/libosp_b200.so

ARCH := -gencode arch=compute_100a,code=sm_100a
# --fmad=false: no FMA contraction anywhere (bit-exact fp32/fp64 rounding)
NVFLAGS := $(ARCH) -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
           -Iinclude -I$(CSRC) --expt-relaxed-constexpr -Xptxas -warn-spills

CU_SRCS := $(CSRC)/kernels/stage.cu $(CSRC)/kernels/resolve.cu $(CSRC)/kernels/elementwise.cu \
           $(CSRC)/kernels/codec.cu $(CSRC)/kernels/stage_tma.cu $(CSRC)/kernels/step_small.cu $(CSRC)/kernels/shard_x.cu $(CSRC)/kernels/shard_chain.cu $(CSRC)/kernels/learner.cu $(CSRC)/capi/osp_capi.cu $(CSRC)/capi/osp_shard.cu $(CSRC)/capi/osp_learner.cu \
           $(CSRC)/capi/osp_codec.cu
CU_OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(CU_SRCS))
HDRS := include/osp_c.h $(CSRC)/osp_internal.h $(CSRC)/kernels/common.cuh $(CSRC)/kernels/tma.cuh $(CSRC)/kernels/shard_common.cuh $(CSRC)/capi/handles.h

# C++ façade of the reference pslab API (include/pslab/*.hpp) over the C-ABI
CXX ?= g++
FACADE := $(PKG)/libpslab_b200.so
FACADE_SRCS := $(wildcard $(CSRC)/pslab/*.cpp)
FACADE_OBJS := $(patsubst $(CSRC)/%.cpp,build/%.o,$(FACADE_SRCS))
FACADE_HDRS := $(wildcard include/pslab/*.hpp) $(CSRC)/pslab/device.hpp include/osp_c.h include/osp_engine.h
CXXFLAGS_FACADE := -std=c++20 -O2 -fPIC -Wall -Wextra -ffp-contract=off -Iinclude -I$(CSRC)/pslab

.PHONY: all lib facade oracle ref dropin clean checked

all: lib facade oracle

lib: $(LIB)

facade: $(FACADE)

build/pslab/%.o: $(CSRC)/pslab/%.cpp $(FACADE_HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS_FACADE) -c $< -o $@

$(FACADE): $(FACADE_OBJS) $(LIB)
	$(CXX) -shared -o $@ $(FACADE_OBJS) -L$(PKG) -losp_b200 -Wl,-rpath,'$$ORIGIN' \
	    -Wl,-soname,libpslab_b200.so

# drop-in proof: the reference harness/tests linked against the façade (needs /root/reference)
dropin: $(FACADE)
	$(MAKE) -C oracle -f Makefile.dropin

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -Xlinker -soname,libosp_b200.so

# checked build: every kernel's indices bounds-checked (OSP_DCHECK, common.cuh);
# the test suite runs against it with OSP_LIB_VARIANT=checked
CHECKED := $(PKG)/libosp_b200_checked.so
CU_OBJS_CHECKED := $(patsubst $(CSRC)/%.cu,build_checked/%.o,$(CU_SRCS))
checked: $(CHECKED)

build_checked/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -DOSP_CHECKED -c $< -o $@

$(CHECKED): $(CU_OBJS_CHECKED)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS_CHECKED) -Xlinker -soname,libosp_b200_checked.so

oracle:
	$(MAKE) -s -C oracle liboracle.so

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf build build_checked $(LIB) $(CHECKED)

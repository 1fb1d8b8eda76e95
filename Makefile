# Builds the framework in-tree (the .so files travel to the GPU box with the
# snapshot):
#   paper_2604_13327_b200/libetgpu.so   C-ABI runtime + sm_100a megakernel + host lowering
#   paper_2604_13327_b200/_etsim*.so    Python module (reference-compatible surface)
PY       ?= python3
CXX      := /usr/bin/g++
NVCC     ?= /usr/local/cuda/bin/nvcc
PKG      := paper_2604_13327_b200
CSRC     := $(PKG)/csrc
BUILD    := build
NLOHMANN ?= $(shell $(PY) -c "import os,sysconfig;print(os.path.join(sysconfig.get_paths()['purelib'],'include','cudnn_frontend','thirdparty','nlohmann'))")
PYBIND   := $(shell $(PY) -c "import pybind11;print(pybind11.get_include())")
PYINC    := $(shell $(PY) -c "import sysconfig;print(sysconfig.get_paths()['include'])")
EXT      := $(shell $(PY) -c "import sysconfig;print(sysconfig.get_config_var('EXT_SUFFIX'))")
ARCH     := -gencode arch=compute_100a,code=sm_100a

CXXFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -Iinclude -I$(NLOHMANN)
NVFLAGS  := -std=c++17 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude -Xptxas -v

HOST_SRCS := symexpr ir materialize sched workloads metrics json_io execute
HOST_OBJS := $(patsubst %,$(BUILD)/host/%.o,$(HOST_SRCS))
CU_OBJS   := $(BUILD)/cu/megakernel.o $(BUILD)/cu/runtime.o
LIB       := $(PKG)/libetgpu.so
MOD       := $(PKG)/_etsim$(EXT)
HDRS      := $(wildcard include/*.h include/etsim/*.hpp $(CSRC)/kernels/*.cuh)

all: $(LIB) $(MOD)

$(BUILD)/host/%.o: $(CSRC)/host/%.cpp $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/cu/megakernel.o: $(CSRC)/kernels/megakernel.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/cu/megakernel.ptxas.txt || (cat $(BUILD)/cu/megakernel.ptxas.txt; false)

$(BUILD)/cu/runtime.o: $(CSRC)/runtime/runtime.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> /dev/null || $(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(HOST_OBJS) $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -cudart static $^ -o $@

$(MOD): $(CSRC)/python/bindings.cpp $(LIB) $(HDRS)
	$(CXX) $(CXXFLAGS) -shared -I$(PYBIND) -I$(PYINC) $< -L$(PKG) -letgpu -Wl,-rpath,'$$ORIGIN' -o $@

clean:
	rm -rf $(BUILD) $(LIB) $(MOD)

.PHONY: all clean

# Top-level build: everything in-tree so the .so files travel with gpurun.
#
#   paper_2211_10017_b200/libmoe_cuda.so       sm_100a kernels + C-ABI (include/moe_cuda.h)
#   paper_2211_10017_b200/libmoeinfer_b200.so  C++ drop-in for the reference's
#                                              moe:: API (include/moeinfer/*.hpp)
#   paper_2211_10017_b200/_moeinfer*.so        pybind11 module, same names as the
#                                              reference's _moeinfer
#   oracle/liboracle.so, oracle/_ref/...       checkers (oracle/Makefile)

NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
PY       ?= python
PKG      := paper_2211_10017_b200
CSRC     := $(PKG)/csrc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -std=c++17 -O3 $(ARCH) -lineinfo --fmad=false -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
            -I$(CSRC) -Iinclude --expt-relaxed-constexpr
CUDA_HOME ?= /usr/local/cuda
CUDA_INC := $(CUDA_HOME)/include
PYINC    := $(shell $(PY) -c "import sysconfig;print(sysconfig.get_paths()['include'])")
PYBIND   := $(shell $(PY) -c "import pybind11;print(pybind11.get_include())")
PYEXT    := $(shell $(PY) -c "import sysconfig;print(sysconfig.get_config_var('EXT_SUFFIX'))")

CU_SRCS  := $(wildcard $(CSRC)/*.cu)
CU_OBJS  := $(patsubst $(CSRC)/%.cu,build/%.o,$(CU_SRCS))
CU_HDRS  := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/moe_cuda.h
HOST_SRCS := $(wildcard $(CSRC)/host/*.cpp)
HOST_HDRS := $(wildcard include/moeinfer/*.hpp) include/moe_cuda.h

LIB_CUDA := $(PKG)/libmoe_cuda.so
LIB_HOST := $(PKG)/libmoeinfer_b200.so
PYMOD    := $(PKG)/_moeinfer$(PYEXT)
BENCHCLI := $(PKG)/moe_bench

.PHONY: all cuda host py tools oracle clean
all: cuda host py tools oracle

cuda: $(LIB_CUDA)
host: $(LIB_HOST)
py: $(PYMOD)
tools: $(BENCHCLI)

build/%.o: $(CSRC)/%.cu $(CU_HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB_CUDA): $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -Xlinker -z,defs -o $@ $(CU_OBJS) -cudart static -lcuda

$(LIB_HOST): $(HOST_SRCS) $(HOST_HDRS) $(LIB_CUDA)
	$(CXX) -std=c++20 -O2 -fPIC -shared -ffp-contract=off -Iinclude -I$(CUDA_INC) \
	  -o $@ $(HOST_SRCS) -L$(PKG) -lmoe_cuda -Wl,-rpath,'$$ORIGIN'

$(PYMOD): $(CSRC)/py_module.cpp $(HOST_HDRS) $(LIB_HOST)
	$(CXX) -std=c++20 -O2 -fPIC -shared -Iinclude -I$(PYINC) -I$(PYBIND) -I$(CUDA_INC) \
	  -o $@ $(CSRC)/py_module.cpp -L$(PKG) -lmoeinfer_b200 -lmoe_cuda -Wl,-rpath,'$$ORIGIN'

# the reference CLI's `moe bench` over a .moec checkpoint's MoE blocks
$(BENCHCLI): $(CSRC)/tools/moe_bench.cpp include/moe_cuda.h $(LIB_CUDA)
	$(CXX) -std=c++17 -O2 -Iinclude -I$(CUDA_INC) -o $@ $(CSRC)/tools/moe_bench.cpp \
	  -L$(PKG) -lmoe_cuda -L$(CUDA_HOME)/lib64 -lcudart -Wl,-rpath,'$$ORIGIN' -Wl,-rpath,$(CUDA_HOME)/lib64

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB_CUDA) $(LIB_HOST) $(PYMOD) $(BENCHCLI)

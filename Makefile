# Build of every native artefact, in-tree (the .so files travel to the GPU box).
#   libsbdt_gpu.so   : sm_100a kernels + the C ABI (include/sbdt_gpu.h)        [product]
#   libsbdt_host.so  : host setup (generators, DT builder, partitioner)        [setup]
#   oracle/liboracle.so : CPU restatement of the path (tests / cpu baseline)   [checker]
#   oracle/_ref/*    : reference sources compiled by path (only where /root/reference exists)
#   $(PKG)/dropin_example : the C++ drop-in headers (include/sbdt/*.hpp) compiled against the
#                      reference's own headers (only where /root/reference exists; header-only
#                      use of the reference types, linked against libsbdt_gpu.so)
PKG      := paper_1902_07554_b200
CSRC     := $(PKG)/csrc
NVCC     ?= nvcc
CXX      ?= g++
# FP64 bit-exactness: no contraction anywhere.
CXXFLAGS := -O3 -std=c++20 -fPIC -ffp-contract=off -Wall -Wextra -Wno-unused-parameter
NVFLAGS  := -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
            -Xcompiler -fPIC -Xcompiler -ffp-contract=off --expt-relaxed-constexpr -Xptxas -v

GPU_SRC  := $(wildcard $(CSRC)/gpu/*.cu)
GPU_HDR  := $(wildcard $(CSRC)/gpu/*.cuh) $(wildcard $(CSRC)/common/*.hpp) include/sbdt_gpu.h
HOST_SRC := $(CSRC)/host/delaunay.cpp $(CSRC)/host/setup.cpp $(CSRC)/host/host_capi.cpp
HOST_HDR := $(wildcard $(CSRC)/host/*.hpp) $(CSRC)/common/predicates.hpp

REF_INC  := /root/reference/proj/include
DROPIN   := $(if $(wildcard $(REF_INC)/sbdt/geometry.hpp),$(PKG)/dropin_example,)

all: $(PKG)/libsbdt_gpu.so $(PKG)/libsbdt_host.so oracle $(DROPIN)

$(PKG)/dropin_example: tests/cpp/dropin_example.cpp include/sbdt/border.hpp include/sbdt/sample_partition.hpp include/sbdt/dc_engine.hpp \
                       include/sbdt_gpu.h $(PKG)/libsbdt_gpu.so
	$(CXX) -O2 -std=c++20 -ffp-contract=off -Iinclude -I$(REF_INC) -o $@ tests/cpp/dropin_example.cpp \
	    -L$(PKG) -lsbdt_gpu -Wl,-rpath,'$$ORIGIN' -lpthread

$(PKG)/libsbdt_host.so: $(HOST_SRC) $(HOST_HDR)
	$(CXX) $(CXXFLAGS) -shared -o $@ $(HOST_SRC) -lpthread

GPU_OBJ  := $(patsubst $(CSRC)/gpu/%.cu,build/gpu/%.o,$(GPU_SRC))

build/gpu/%.o: $(CSRC)/gpu/%.cu $(GPU_HDR)
	@mkdir -p build/gpu
	$(NVCC) $(NVFLAGS) -Iinclude -c -o $@ $< 2> build/gpu/$*.ptxas.log || (cat build/gpu/$*.ptxas.log; exit 1)

$(PKG)/libsbdt_gpu.so: $(GPU_OBJ)
	$(NVCC) -shared -gencode arch=compute_100a,code=sm_100a -o $@ $(GPU_OBJ)
	cat build/gpu/*.ptxas.log > $(PKG)/ptxas.log

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(PKG)/*.so $(PKG)/ptxas.log $(PKG)/dropin_example build/gpu
	$(MAKE) -C oracle clean

.PHONY: all oracle clean

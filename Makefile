# Builds the product library (sm_100a) and the CPU oracle (test infrastructure).
NVCC    ?= nvcc
ARCH    ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC,-Wall -Iinclude -Xptxas -v $(EXTRA)
PKG      = paper_2308_03121_b200
SRC      = $(PKG)/csrc/nnvisr.cpp $(PKG)/csrc/kernels.cu $(PKG)/csrc/kernels_tma.cu $(PKG)/csrc/kernels_yuv.cu $(PKG)/csrc/scene.cu
HDR      = include/nnvisr.h $(PKG)/csrc/internal.h $(PKG)/csrc/common.cuh
LIB      = $(PKG)/libnnvisr.so
ORACLE   = oracle/liboracle.so

all: $(LIB) $(ORACLE)

$(PKG)/build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p $(PKG)/build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(PKG)/build/$*.ptxas.txt || (cat $(PKG)/build/$*.ptxas.txt; false)

$(PKG)/build/%.o: $(PKG)/csrc/%.cpp $(HDR)
	@mkdir -p $(PKG)/build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(PKG)/build/nnvisr.o $(PKG)/build/kernels.o $(PKG)/build/kernels_tma.o $(PKG)/build/kernels_yuv.o $(PKG)/build/scene.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static

$(ORACLE): oracle/nnvisr_oracle.c
	gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -Wall -fPIC -shared -o $@ $< -lm

clean:
	rm -rf $(PKG)/build $(LIB) $(ORACLE)

.PHONY: all clean

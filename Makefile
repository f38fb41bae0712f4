# Builds the product library (sm_100a) and the CPU oracle (test infrastructure).
NVCC    ?= nvcc
ARCH    ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC,-Wall -Iinclude -Xptxas -v $(EXTRA)
PKG      = paper_2308_03121_b200
SRC      = $(PKG)/csrc/nnvisr.cpp $(PKG)/csrc/comm.cpp $(PKG)/csrc/kernels.cu $(PKG)/csrc/kernels_tma.cu $(PKG)/csrc/kernels_yuv.cu $(PKG)/csrc/scene.cu $(PKG)/csrc/kernels_strip.cu
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

$(LIB): $(PKG)/build/nnvisr.o $(PKG)/build/comm.o $(PKG)/build/kernels.o $(PKG)/build/kernels_tma.o $(PKG)/build/kernels_yuv.o $(PKG)/build/scene.o $(PKG)/build/kernels_strip.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static -ldl

$(ORACLE): oracle/nnvisr_oracle.c
	gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -Wall -fPIC -shared -o $@ $< -lm

# checked build (device-side bounds checks, -DNNVISR_CHECKED): select it with
# NNVISR_LIBNAME=libnnvisr_checked.so (tools/checked_tests.sh)
CHK      = $(PKG)/libnnvisr_checked.so
checked: $(CHK)

$(PKG)/build_checked/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p $(PKG)/build_checked
	$(NVCC) $(NVFLAGS) -DNNVISR_CHECKED -c $< -o $@ 2> $(PKG)/build_checked/$*.ptxas.txt || (cat $(PKG)/build_checked/$*.ptxas.txt; false)

$(PKG)/build_checked/%.o: $(PKG)/csrc/%.cpp $(HDR)
	@mkdir -p $(PKG)/build_checked
	$(NVCC) $(NVFLAGS) -DNNVISR_CHECKED -c $< -o $@

$(CHK): $(PKG)/build_checked/nnvisr.o $(PKG)/build_checked/comm.o $(PKG)/build_checked/kernels.o $(PKG)/build_checked/kernels_tma.o $(PKG)/build_checked/kernels_yuv.o $(PKG)/build_checked/scene.o $(PKG)/build_checked/kernels_strip.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static -ldl

clean:
	rm -rf $(PKG)/build $(PKG)/build_checked $(LIB) $(CHK) $(ORACLE)

.PHONY: all checked clean

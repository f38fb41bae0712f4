# build libnnvisr_<tag>.so with kernels_strip.cu compiled with extra flags (A/B experiments):
# bash tools/build_variant.sh s4 -DNNVISR_STRIP_STAGES=4
tag=$1; shift
P=paper_2308_03121_b200
mkdir -p $P/build_$tag
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-Wall -Iinclude "$@" \
  -c $P/csrc/kernels_strip.cu -o $P/build_$tag/kernels_strip.o || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/libnnvisr_$tag.so \
  $(ls $P/build/*.o | grep -v kernels_strip.o) $P/build_$tag/kernels_strip.o -cudart static -ldl

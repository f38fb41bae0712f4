#!/bin/bash
# f2t bottleneck probe: NNVISR_F2T_DEBUG 1 = no conversion, 2 = no stores, 4 = no loads.  The switches
# exist only in an experiments build (-DNNVISR_EXPERIMENTS), built here as libnnvisr_x.so.
make -C "$(dirname "$0")/.." -j8 all >/dev/null || exit 1
P=paper_2308_03121_b200
mkdir -p /tmp/nnvisr_x && for f in nnvisr.cpp kernels.cu kernels_tma.cu kernels_yuv.cu scene.cu; do
  nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Iinclude \
       -DNNVISR_EXPERIMENTS -c $P/csrc/$f -o /tmp/nnvisr_x/${f%.*}.o || exit 1; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/libnnvisr_x.so /tmp/nnvisr_x/*.o -cudart static || exit 1
for args in "--workload c4" "--workload c4 --f2t-mode batch" "--workload c2 --f2t-mode store" "--workload c2"; do
 for dbg in 0 1 2 4; do
  NNVISR_LIBNAME=libnnvisr_x.so NNVISR_F2T_DEBUG=$dbg timeout 300 python bench.py $args --frames 240 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/pr.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/pr.log').read().strip().splitlines()[-1]); v=d['per_direction']['f2t']; print('$args dbg $dbg', round(v['achieved_gbs']))"
 done
done

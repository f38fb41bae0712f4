#!/bin/bash
# Every bench workload / mode once (default steps), one JSON line each into gpurun_out/all/.
mkdir -p gpurun_out/all
python bench.py > gpurun_out/all/c2.json 2> gpurun_out/all/c2.err
for wl in c3 c4 c5 c1; do python bench.py --workload $wl --no-cpu-baseline > gpurun_out/all/$wl.json 2> gpurun_out/all/$wl.err; done
python bench.py --workload c2 --f2t-mode store --no-e2e --no-cpu-baseline > gpurun_out/all/c2_store.json 2>/dev/null
python bench.py --workload c5 --f2t-mode store --no-e2e --no-cpu-baseline > gpurun_out/all/c5_store.json 2>/dev/null
python bench.py --workload c4 --f2t-mode batch --no-e2e --no-cpu-baseline > gpurun_out/all/c4_batch.json 2>/dev/null
python bench.py --workload c4 --emit --no-e2e --no-cpu-baseline > gpurun_out/all/c4_emit.json 2>/dev/null
python bench.py --workload c1 --emit --no-e2e --no-cpu-baseline > gpurun_out/all/c1_emit.json 2>/dev/null
python bench.py --workload c1 --graph --no-e2e --no-cpu-baseline > gpurun_out/all/c1_graph.json 2>/dev/null
python bench.py --workload c2 --detect --no-e2e --no-cpu-baseline > gpurun_out/all/c2_detect.json 2>/dev/null
for wl in c2 c3 c4 c5; do python bench.py --workload $wl --tensors yuv --no-e2e --no-cpu-baseline > gpurun_out/all/${wl}_yuv.json 2>/dev/null; done
for wl in c2 c4; do python bench.py --workload $wl --chroma-loc left --no-e2e --no-cpu-baseline > gpurun_out/all/${wl}_left.json 2>/dev/null; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/all/reference_c2.json 2>/dev/null

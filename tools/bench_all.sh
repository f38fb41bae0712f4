#!/bin/bash
# Every bench workload / mode once (default steps), one JSON line each into gpurun_out/all/ (round 2 flags).
mkdir -p gpurun_out/all
Q="--per-config '' --no-compare-modes"
run() { name=$1; shift; eval python bench.py "$@" $Q > gpurun_out/all/$name.json 2> gpurun_out/all/$name.err; }
run c5 --workload c5
run c5_mat --workload c5 --f2t-mode materialize --no-e2e --no-cpu-baseline
run c2 --workload c2
run c2_mat --workload c2 --f2t-mode materialize --no-e2e --no-cpu-baseline
run c3 --workload c3
run c3_mat --workload c3 --f2t-mode materialize --no-e2e --no-cpu-baseline
run c4 --workload c4
run c4_mat --workload c4 --f2t-mode materialize --no-e2e --no-cpu-baseline
run c4_batch --workload c4 --f2t-mode batch --no-e2e --no-cpu-baseline
run c4_emit --workload c4 --emit --no-e2e --no-cpu-baseline
run c1 --workload c1
run c1_graph --workload c1 --graph --no-e2e --no-cpu-baseline
run c1_emit --workload c1 --emit --no-e2e --no-cpu-baseline
run c2_detect --workload c2 --detect --no-e2e --no-cpu-baseline
for wl in c2 c3 c4 c5; do run ${wl}_yuv --workload $wl --tensors yuv --f2t-mode materialize --no-e2e --no-cpu-baseline; done
for wl in c2 c4; do run ${wl}_left --workload $wl --chroma-loc left --no-e2e --no-cpu-baseline; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/all/reference_c5.json 2>/dev/null
python bench.py --impl reference --workload c2 --steps 2 --warmup 1 > gpurun_out/all/reference_c2.json 2>/dev/null

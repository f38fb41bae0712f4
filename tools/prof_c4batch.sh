mkdir -p gpurun_out/prof3
B="python bench.py --workload c4 --f2t-mode batch --frames 240 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config '' --no-compare-modes"
eval $B > gpurun_out/prof3/plain.json 2>&1 || exit 1
eval ncu --set full --clock-control none --import-source on -k regex:strip -s 2 -c 1 -o gpurun_out/prof3/c4batch_strip $B > gpurun_out/prof3/n1.log 2>&1

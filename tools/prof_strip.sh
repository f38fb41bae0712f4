# ncu --set full of the strip kernel in c2 store mode (one launch) + c4 materialised
mkdir -p gpurun_out/prof2
B="python bench.py --workload c2 --f2t-mode store --frames 120 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --per-config ''"
eval $B > gpurun_out/prof2/plain.json 2>&1 || exit 1
eval ncu --set full --clock-control none --import-source on -k regex:strip -c 1 -o gpurun_out/prof2/strip_c2store $B > gpurun_out/prof2/n1.log 2>&1

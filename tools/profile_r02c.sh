#!/bin/bash
# Round-2 final profile capture (after the strip rewrite and the launch-size changes):
#  1. the default bench command, short, exits 0 without ncu
#  2. its launch list (our kernels): ncu --metrics gpu__time_duration.sum + dram bytes
#  3. ncu --set full of one launch each: t2f_tma (c5, 52 tuples), f2t_strip420 (c5 store, 80-frame
#     region), f2t_tma (c5 materialised), f2t_strip420 (c2 store), f2t_tma (c4 materialised)
mkdir -p gpurun_out/prof_c
PART=${1:-a}  # a: launch list, t2f, strip (c5, c2); b: f2t_tma (c5 materialised, c4) -- two calls, each under 64 MiB of output
if [ $PART = a ]; then
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config '' --no-compare-modes"
eval $B > gpurun_out/prof_c/plain.json 2> gpurun_out/prof_c/plain.err || exit 1
eval ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k "'regex:f2t|t2f|sad|cut_kernel|copy'" --log-file gpurun_out/prof_c/launches_r02c.csv $B > gpurun_out/prof_c/ncu_launch.log 2>&1
C5="python bench.py --frames 256 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config '' --no-compare-modes"
eval ncu --set full --clock-control none --import-source on -k regex:t2f_tma -s 2 -c 1 -o gpurun_out/prof_c/r02c_c5_t2f_full $C5 > gpurun_out/prof_c/n1.log 2>&1
eval ncu --set full --clock-control none --import-source on -k regex:f2t_strip -s 1 -c 1 -o gpurun_out/prof_c/r02c_c5store_strip_full $C5 > gpurun_out/prof_c/n2.log 2>&1
fi
if [ $PART = b ]; then
C5="python bench.py --frames 256 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config '' --no-compare-modes"
eval ncu --set full --clock-control none --import-source on -k regex:f2t_tma -s 2 -c 1 -o gpurun_out/prof_c/r02c_c5mat_f2t_full $C5 --f2t-mode materialize > gpurun_out/prof_c/n3.log 2>&1
fi
if [ $PART = a ]; then
C2="python bench.py --workload c2 --frames 120 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config '' --no-compare-modes"
eval ncu --set full --clock-control none --import-source on -k regex:f2t_strip -s 1 -c 1 -o gpurun_out/prof_c/r02c_c2store_strip_full $C2 > gpurun_out/prof_c/n4.log 2>&1
fi
if [ $PART = b ]; then
C4="python bench.py --workload c4 --frames 240 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config '' --no-compare-modes"
eval ncu --set full --clock-control none --import-source on -k regex:f2t_tma -s 2 -c 1 -o gpurun_out/prof_c/r02c_c4_f2t_full $C4 > gpurun_out/prof_c/n5.log 2>&1
fi
du -sh gpurun_out/prof_c; ls -la gpurun_out/prof_c

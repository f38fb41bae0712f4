#!/bin/bash
# Round-2 refresh after the dynamic-tile strip kernel and the NARROW TMA variant (one GPU):
# launch list of the default bench command, ncu --set full of the strip kernel (c5 store, c2 store,
# c4 batches) and of the NARROW f2t_tma (c4 2-frame windows)
mkdir -p gpurun_out/prof4
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config '' --no-compare-modes"
eval $B > gpurun_out/prof4/plain.json 2>&1 || exit 1
eval ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k "'regex:f2t|t2f|sad|cut_kernel'" --log-file gpurun_out/prof4/launches_r02.csv $B > gpurun_out/prof4/ncu_launch.log 2>&1
C5="python bench.py --frames 256 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config '' --no-compare-modes"
eval ncu --set full --clock-control none --import-source on -k regex:f2t_strip -s 2 -c 1 -o gpurun_out/prof4/r02_c5store_strip_full $C5 > gpurun_out/prof4/n2.log 2>&1
C2="python bench.py --workload c2 --frames 160 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config '' --no-compare-modes"
eval ncu --set full --clock-control none --import-source on -k regex:f2t_strip -s 1 -c 1 -o gpurun_out/prof4/r02_c2store_strip_full $C2 > gpurun_out/prof4/n4.log 2>&1
C4B="python bench.py --workload c4 --f2t-mode batch --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config '' --no-compare-modes"
eval ncu --set full --clock-control none --import-source on -k regex:f2t_strip -s 2 -c 1 -o gpurun_out/prof4/r02_c4batch_strip_full $C4B > gpurun_out/prof4/n5.log 2>&1
C4="python bench.py --workload c4 --frames 240 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config '' --no-compare-modes"
eval ncu --set full --clock-control none --import-source on -k regex:f2t_tma -s 2 -c 1 -o gpurun_out/prof4/r02_c4_f2t_full $C4 > gpurun_out/prof4/n6.log 2>&1
du -sh gpurun_out/prof4

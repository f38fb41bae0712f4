mkdir -p gpurun_out/prof
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config '' --no-compare-modes"
eval ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k "'regex:f2t|t2f|sad|cut_kernel'" --log-file gpurun_out/prof/launches_r02.csv $B > gpurun_out/prof/ncu_launch.log 2>&1
wc -l gpurun_out/prof/launches_r02.csv

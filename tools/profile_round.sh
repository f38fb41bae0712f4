#!/bin/bash
# Round profile capture (run on the GPU box; keep gpurun_out under 64 MiB): PART=c2 -> launch list of
# our kernels + ncu --set full of t2f and f2t at c2; PART=c5 -> the same two captures at c5.
mkdir -p gpurun_out/prof
if [ "${PART:-c2}" = c2 ]; then
  B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
  $B > gpurun_out/prof/plain.json 2>&1 || exit 1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      -k regex:"f2t|t2f|sad|cut_kernel" --log-file gpurun_out/prof/launches_r01.csv $B > gpurun_out/prof/ncu_launch.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:t2f_tma -s 3 -c 1 -o gpurun_out/prof/r01_t2f_full $B > gpurun_out/prof/n1.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:f2t_tma -s 3 -c 1 -o gpurun_out/prof/r01_f2t_full $B > gpurun_out/prof/n2.log 2>&1
else
  C5="python bench.py --workload c5 --frames 64 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  ncu --set full --clock-control none --import-source on -k regex:f2t_tma -s 3 -c 1 -o gpurun_out/prof/r01_c5_f2t_full $C5 > gpurun_out/prof/n3.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:t2f_tma -s 3 -c 1 -o gpurun_out/prof/r01_c5_t2f_full $C5 > gpurun_out/prof/n4.log 2>&1
fi
du -sh gpurun_out

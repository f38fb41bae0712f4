#!/bin/bash
# Generic tuning sweep: tools/sweep.sh DIR "wl1 wl2 ..." "ENV=.. ENV=..;ENV=..;..." [frames]
# Prints, per workload and env setting, the direction's TB/s and fraction of the measured peak.
dir=$1; wls=$2; cfgs=$3; frames=${4:-0}
IFS=';' read -ra CF <<< "$cfgs"
for wl in $wls; do
 for cfg in "${CF[@]}"; do
  env $cfg timeout 300 python bench.py --workload $wl --frames $frames --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/sw.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); v=d['per_direction']['$dir']; print('$wl $cfg', round(v['achieved_gbs']), round(v['frac_of_measured_peak'],3))" 2>&1 | tail -1
 done
done

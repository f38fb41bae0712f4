#!/bin/bash
# tools/ab_env.sh DIR "workloads" frames rounds "ENV1" "ENV2" ... -- same-box A/B of env settings (lib via NNVISR_LIBNAME in the env string)
dir=$1; wls=$2; frames=${3:-240}; rounds=${4:-2}; shift 4
for wl in $wls; do
 for r in $(seq $rounds); do
  for cfg in "$@"; do
   env $cfg timeout 300 python bench.py --workload $wl --frames $frames --steps 5 --warmup 2 --no-cpu-baseline --no-e2e $EXTRA > gpurun_out/ab.log 2>&1
   python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); v=d['per_direction']['$dir']; print('$wl [$cfg]', round(v['achieved_gbs']), round(v['frac_of_measured_peak'],3))" 2>&1 | tail -1
  done
 done
done

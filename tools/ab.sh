#!/bin/bash
# A/B on one box: tools/ab.sh DIR "workloads" frames rounds lib1 lib2 ... -- alternates in-tree builds
# (paper_2308_03121_b200/<lib>) so box-to-box variance cancels.  Prints DIR TB/s per run.
dir=$1; wls=$2; frames=${3:-240}; rounds=${4:-2}; shift 4; libs=${@:-libnnvisr_a.so libnnvisr.so}
for wl in $wls; do
 for r in $(seq $rounds); do
  for lib in $libs; do
   NNVISR_LIBNAME=$lib timeout 300 python bench.py --workload $wl --frames $frames --steps 5 --warmup 2 --no-cpu-baseline --no-e2e $EXTRA > gpurun_out/ab.log 2>&1
   python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); v=d['per_direction']['$dir']; print('$wl $lib', round(v['achieved_gbs']), round(v['frac_of_measured_peak'],3))" 2>&1 | tail -1
  done
 done
done

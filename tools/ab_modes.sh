#!/bin/bash
# Same-box A/B over bench modes: tools/ab_modes.sh "lib1 lib2" "wl:mode wl:mode ..." [rounds]
libs=$1; specs=$2; rounds=${3:-2}
for r in $(seq $rounds); do
 for lib in $libs; do
  for spec in $specs; do wl=${spec%%:*}; mode=${spec##*:}
   NNVISR_LIBNAME=$lib python bench.py --workload $wl --frames 240 --f2t-mode $mode --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/x.json 2>/dev/null
   python -c "
import json;d=json.load(open('gpurun_out/x.json'));v=d['per_direction']['f2t']; print('$lib $wl $mode', round(v['achieved_gbs']), round(v['fps']))"
  done
 done
done

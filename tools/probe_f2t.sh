#!/bin/bash
# f2t bottleneck probe: NNVISR_F2T_DEBUG 1 = no conversion, 2 = no stores, 4 = no loads (experiments only)
for args in "--workload c4" "--workload c4 --f2t-mode batch" "--workload c2 --f2t-mode store" "--workload c2"; do
 for dbg in 0 1 2 4; do
  NNVISR_F2T_DEBUG=$dbg timeout 300 python bench.py $args --frames 240 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/pr.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/pr.log').read().strip().splitlines()[-1]); v=d['per_direction']['f2t']; print('$args dbg $dbg', round(v['achieved_gbs']))"
 done
done

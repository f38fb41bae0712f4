# t2f_tma tuning sweep: input stages S and smem budget (CTAs per SM)
for wl in c2 c4 c3; do
 for cfg in "3 72" "2 72" "4 100" "6 150" "8 200" "4 227" "5 150"; do
  set -- $cfg
  NNVISR_T2F_STAGES=$1 NNVISR_T2F_SMEM_KB=$2 timeout 300 python bench.py --workload $wl --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/sw.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); v=d['per_direction']['t2f']; print('$wl st=$1 smem=$2', round(v['achieved_gbs']), round(v['frac_of_measured_peak'],3))" 2>&1 | tail -1
 done
done

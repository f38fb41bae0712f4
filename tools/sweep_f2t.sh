# f2t_tma tuning sweep: band height B, output buffers, input stages (smem up to 227 KB)
for wl in c2 c4 c5s c3; do
 for cfg in "1 3 2" "1 6 2" "2 2 2" "2 3 2" "2 4 2" "3 2 2" "3 3 2" "4 2 2" "4 3 1" "2 2 3"; do
  set -- $cfg
  if [ $wl = c5s ]; then W="--workload c5 --scaling weak"; else W="--workload $wl"; fi
  NNVISR_F2T_BAND=$1 NNVISR_F2T_NOB=$2 NNVISR_F2T_STAGES=$3 NNVISR_F2T_SMEM_KB=227 timeout 300 python bench.py $W --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/sw.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); v=d['per_direction']['f2t']; print('$wl band=$1 nob=$2 st=$3', round(v['achieved_gbs']), round(v['frac_of_measured_peak'],3))" 2>&1 | tail -1
 done
done

for wl in c4 c2; do
for cfg in "" "NNVISR_F2T_BAND=4" "NNVISR_F2T_BAND=4 NNVISR_F2T_NOB=3" "NNVISR_F2T_NOB=3" "NNVISR_F2T_NOB=4" "NNVISR_F2T_LOADER=1 NNVISR_F2T_RELFIRST=0 NNVISR_F2T_NOB=3" "NNVISR_F2T_BAND=4 NNVISR_F2T_LOADER=1 NNVISR_F2T_RELFIRST=0 NNVISR_F2T_NOB=3"; do
 env $cfg timeout 300 python bench.py --workload $wl --frames 240 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --tensors yuv > gpurun_out/sw.log 2>&1
 python -c "
import json; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); v=d['per_direction']['f2t']; print('$wl [$cfg]', round(v['achieved_gbs']))"
done; done

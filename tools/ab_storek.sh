# store-ring region size A/B (frames per region) on c5 (1024 frames) and c2
out=gpurun_out/ab_storek; mkdir -p $out
for rep in 1 2; do for k in 0 80 160 320; do
 python bench.py --workload c5 --frames 1024 --store-k $k --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c5_k${k}_$rep.json 2>&1
done; for k in 0 240; do
 python bench.py --workload c2 --store-k $k --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c2_k${k}_$rep.json 2>&1
done; done
python tools/show_ab.py $out | sort
for f in $out/*.json; do python -c "
import json,sys; d=json.loads([l for l in open('$f') if l.startswith('{')][-1]); pd=d['per_direction']; print('$f'.split('/')[-1], {k:round(v['ms_per_step'],2) for k,v in pd.items()}, round(d['ms_per_step'],2))"; done

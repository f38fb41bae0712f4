# t2f tuples-per-launch A/B on c5 (1024 frames) and c2
out=gpurun_out/ab_t2fchunk; mkdir -p $out
for rep in 1 2; do for k in 0 26 52; do
 python bench.py --workload c5 --frames 1024 --t2f-chunk $k --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c5_t${k}_$rep.json 2>&1
 python bench.py --workload c2 --t2f-chunk $k --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c2_t${k}_$rep.json 2>&1
done; done
python tools/show_ab.py $out | sort

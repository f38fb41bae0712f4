# paper-grouping n = 1 workloads (c4, c1) in store mode on the padded layout vs materialised / Fig. 1 batches
out=gpurun_out/ab_c4store; mkdir -p $out
for rep in 1 2; do for m in store materialize batch; do
 python bench.py --workload c4 --f2t-mode $m --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c4_${m}_$rep.json 2>&1
 python bench.py --workload c1 --f2t-mode $m --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c1_${m}_$rep.json 2>&1
done; done
python tools/show_ab.py $out | sort

# store ring layout A/B: scene-padded (every tuple a window) vs one slot per frame (+ materialised edge tuples)
out=gpurun_out/ab_layout; mkdir -p $out
python -m pytest tests/test_gpu_store_ring.py tests/test_gpu_bench_shards.py -q -x > $out/tests.txt 2>&1; echo rc=$? >> $out/tests.txt; tail -2 $out/tests.txt
for rep in 1 2; do for lay in padded frames; do
 python bench.py --workload c5 --frames 1024 --store-layout $lay --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c5_${lay}_$rep.json 2>&1
 python bench.py --workload c2 --store-layout $lay --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c2_${lay}_$rep.json 2>&1
 python bench.py --workload c3 --store-layout $lay --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c3_${lay}_$rep.json 2>&1
done; done
python bench.py --workload c2 --detect --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c2_detect_padded.json 2>&1
python tools/show_ab.py $out | sort

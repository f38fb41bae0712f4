out=gpurun_out/${1:-abc4b}; mkdir -p $out
for rep in 1 2; do for lib in ${LIBS:-libnnvisr_a.so libnnvisr_b.so}; do
 NNVISR_LIBNAME=$lib python bench.py --workload c4 --f2t-mode batch --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c4_batch_${lib%.so}_$rep.json 2>&1
done; done
for t in 6 12 24; do NNVISR_F2T_STRIP_TPC=$t python bench.py --workload c4 --f2t-mode batch --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c4_batch_tpc$t.json 2>&1; done
for t in 6 24; do NNVISR_F2T_STRIP_TPC=$t python bench.py --workload c2 --f2t-mode store --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c2_store_tpc$t.json 2>&1; done

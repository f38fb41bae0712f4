# strip-kernel decomposition (experiments): loads off / stores off / both, c5 and c2 store mode (f2t timing only)
out=gpurun_out/ab_decomp; mkdir -p $out
for rep in 1 2; do for lib in libnnvisr.so libnnvisr_nostore.so libnnvisr_noload.so libnnvisr_noboth.so; do
 NNVISR_LIBNAME=$lib python bench.py --workload c5 --frames 1024 --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c5_${lib%.so}_$rep.json 2>&1
 NNVISR_LIBNAME=$lib python bench.py --workload c4 --f2t-mode batch --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c4b_${lib%.so}_$rep.json 2>&1
done; done
python tools/show_ab.py $out | sort

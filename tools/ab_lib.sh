# same-box A/B of two library builds: LIBS="libnnvisr.so libnnvisr_b.so" bash tools/ab_lib.sh <outdir>
out=gpurun_out/${1:-ab}
mkdir -p $out
python -m pytest tests/test_gpu_strip.py tests/test_gpu_store_ring.py -q -x > $out/tests.txt 2>&1 || { tail -30 $out/tests.txt; exit 1; }
for rep in 1 2; do
for lib in ${LIBS:-libnnvisr.so libnnvisr_b.so}; do
 tag=${lib%.so}_$rep
 NNVISR_LIBNAME=$lib python bench.py --workload c2 --f2t-mode store --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c2_store_$tag.json 2>&1
 NNVISR_LIBNAME=$lib python bench.py --workload c5 --frames 1024 --f2t-mode store --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c5_store_$tag.json 2>&1
 NNVISR_LIBNAME=$lib python bench.py --workload c4 --f2t-mode batch --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c4_batch_$tag.json 2>&1
 NNVISR_F2T_STRIP=1 NNVISR_LIBNAME=$lib python bench.py --workload c4 --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c4_strip_$tag.json 2>&1
done
done

# same-box A/B of the strip kernel: tests on the new build (+ checked), then
# store / batch benches for LIBS (default: libnnvisr.so libnnvisr_old.so)
out=gpurun_out/${1:-ab_r02s}
mkdir -p $out
python -m pytest tests/test_gpu_strip.py tests/test_gpu_store_ring.py tests/test_gpu_batch_store.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > $out/tests.txt 2>&1 || { tail -30 $out/tests.txt; exit 1; }
NNVISR_LIBNAME=libnnvisr_checked.so python -m pytest tests/test_gpu_strip.py tests/test_gpu_store_ring.py -q -x > $out/tests_checked.txt 2>&1 || { tail -30 $out/tests_checked.txt; exit 1; }
for rep in 1 2; do
for lib in ${LIBS:-libnnvisr.so libnnvisr_old.so}; do
 tag=${lib%.so}_$rep
 NNVISR_LIBNAME=$lib python bench.py --workload c2 --f2t-mode store --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c2_store_$tag.json 2>&1
 NNVISR_LIBNAME=$lib python bench.py --workload c5 --frames 1024 --f2t-mode store --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c5_store_$tag.json 2>&1
 NNVISR_LIBNAME=$lib python bench.py --workload c4 --f2t-mode batch --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c4_batch_$tag.json 2>&1
done
done
python tools/show_ab.py $out > $out/summary.txt 2>&1; cat $out/summary.txt

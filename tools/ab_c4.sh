# same-box A/B (c4 materialised + c4 emit) of libnnvisr_a.so vs libnnvisr_b.so
out=gpurun_out/${1:-abc4}; mkdir -p $out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x > $out/tests.txt 2>&1 || { tail -20 $out/tests.txt; exit 1; }
for rep in 1 2; do for lib in libnnvisr_a.so libnnvisr_b.so; do
 NNVISR_LIBNAME=$lib python bench.py --workload c4 --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c4_${lib%.so}_$rep.json 2>&1
 NNVISR_LIBNAME=$lib python bench.py --workload c4 --emit --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c4emit_${lib%.so}_$rep.json 2>&1
done; done

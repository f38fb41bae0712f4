# same-box A/B of the t2f kernel (libnnvisr_a.so vs libnnvisr_b.so) on c5 / c2 / c4 / c3, tests first
out=gpurun_out/${1:-abt2f}; mkdir -p $out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_next3.py -q -x > $out/tests.txt 2>&1 || { tail -20 $out/tests.txt; exit 1; }
for rep in 1 2; do for lib in libnnvisr_a.so libnnvisr_b.so; do
 for wl in c5 c2 c4 c3; do
  NNVISR_LIBNAME=$lib python bench.py --workload $wl --frames 480 --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/${wl}_${lib%.so}_$rep.json 2>&1
 done
done; done

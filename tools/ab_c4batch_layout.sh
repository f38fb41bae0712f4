out=gpurun_out/ab4; mkdir -p $out
NNVISR_LIBNAME=libnnvisr_l160.so python -m pytest tests/test_gpu_batch_store.py -q -x -k "not full" > $out/t.txt 2>&1
for rep in 1 2 3; do for lib in libnnvisr.so libnnvisr_l160.so libnnvisr_old.so; do
 NNVISR_LIBNAME=$lib python bench.py --workload c4 --f2t-mode batch --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c4_batch_${lib%.so}_$rep.json 2>&1
done; done
python tools/show_ab.py $out | sort

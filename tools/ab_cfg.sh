# same-box A/B of environment configurations on the strip-kernel workloads:
# CFGS="new: old:NNVISR_LIBNAME=libnnvisr_old.so tpc6:NNVISR_F2T_STRIP_TPC=6" bash tools/ab_cfg.sh <outdir> [reps]
out=gpurun_out/${1:-ab_cfg}
reps=${2:-2}
mkdir -p $out
python -m pytest tests/test_gpu_strip.py tests/test_gpu_store_ring.py tests/test_gpu_batch_store.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > $out/tests.txt 2>&1 || { tail -30 $out/tests.txt; exit 1; }
NNVISR_LIBNAME=libnnvisr_checked.so python -m pytest tests/test_gpu_strip.py tests/test_gpu_store_ring.py -q -x > $out/tests_checked.txt 2>&1 || { tail -30 $out/tests_checked.txt; exit 1; }
for rep in $(seq $reps); do
for cfg in $CFGS; do
 name=${cfg%%:*}; envs=${cfg#*:}; envs=${envs//,/ }
 env $envs python bench.py --workload c2 --f2t-mode store --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c2_store_${name}_$rep.json 2>&1
 env $envs python bench.py --workload c5 --frames 1024 --f2t-mode store --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c5_store_${name}_$rep.json 2>&1
 env $envs python bench.py --workload c4 --f2t-mode batch --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c4_batch_${name}_$rep.json 2>&1
done
done
python tools/show_ab.py $out > $out/summary.txt 2>&1; cat $out/summary.txt

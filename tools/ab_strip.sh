mkdir -p gpurun_out/b2
python -m pytest tests/test_gpu_strip.py tests/test_gpu_store_ring.py -q -x > gpurun_out/b2/tests.txt 2>&1
B="python bench.py --per-config '' --no-e2e --no-cpu-baseline"
for s in 1 0; do
 NNVISR_F2T_STRIP=$s python bench.py --workload c2 --f2t-mode store --per-config "" --no-e2e --no-cpu-baseline > gpurun_out/b2/c2_store_$s.json 2>&1
 NNVISR_F2T_STRIP=$s python bench.py --workload c4 --per-config "" --no-e2e --no-cpu-baseline > gpurun_out/b2/c4_$s.json 2>&1
 NNVISR_F2T_STRIP=$s python bench.py --workload c4 --f2t-mode batch --per-config "" --no-e2e --no-cpu-baseline > gpurun_out/b2/c4_batch_$s.json 2>&1
 NNVISR_F2T_STRIP=$s python bench.py --workload c5 --f2t-mode store --frames 1024 --per-config "" --no-e2e --no-cpu-baseline > gpurun_out/b2/c5_store_$s.json 2>&1
done
for r in 8 16 64; do NNVISR_F2T_STRIP_ROWS=$r python bench.py --workload c2 --f2t-mode store --per-config "" --no-e2e --no-cpu-baseline > gpurun_out/b2/c2_store_rows$r.json 2>&1; done

mkdir -p gpurun_out/b9
python -m pytest tests/test_gpu_strip.py tests/test_gpu_store_ring.py -q -x > gpurun_out/b9/tests.txt 2>&1 || { tail -30 gpurun_out/b9/tests.txt; exit 1; }
for s in 1; do
 NNVISR_F2T_STRIP=$s python bench.py --workload c2 --f2t-mode store --per-config "" --no-e2e --no-cpu-baseline > gpurun_out/b9/c2_store_$s.json 2>&1
 NNVISR_F2T_STRIP=$s python bench.py --workload c4 --per-config "" --no-e2e --no-cpu-baseline > gpurun_out/b9/c4_$s.json 2>&1
 NNVISR_F2T_STRIP=$s python bench.py --workload c4 --f2t-mode batch --per-config "" --no-e2e --no-cpu-baseline > gpurun_out/b9/c4_batch_$s.json 2>&1
 NNVISR_F2T_STRIP=$s python bench.py --workload c5 --f2t-mode store --frames 1024 --per-config "" --no-e2e --no-cpu-baseline > gpurun_out/b9/c5_store_$s.json 2>&1
done
B="python bench.py --workload c2 --f2t-mode store --frames 120 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --per-config ''"
eval ncu --set full --clock-control none --import-source on -k regex:strip -c 1 -o gpurun_out/b9/strip_c2store $B > gpurun_out/b9/n1.log 2>&1

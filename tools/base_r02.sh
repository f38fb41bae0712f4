mkdir -p gpurun_out/base
for a in "c2" "c5" "c4"; do python bench.py --workload $a --no-e2e --no-cpu-baseline > gpurun_out/base/$a.json 2> gpurun_out/base/$a.err; done
python bench.py --workload c2 --f2t-mode store --no-e2e --no-cpu-baseline > gpurun_out/base/c2_store.json 2>gpurun_out/base/c2_store.err
python bench.py --workload c4 --f2t-mode batch --no-e2e --no-cpu-baseline > gpurun_out/base/c4_batch.json 2>gpurun_out/base/c4_batch.err
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/base/smi.txt

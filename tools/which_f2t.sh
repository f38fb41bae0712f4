mkdir -p gpurun_out/r2c
timeout -s KILL 300 python -m pytest tests/test_gpu_shards.py tests/test_gpu_comm.py -q -x > gpurun_out/r2c/tests.txt 2>&1; echo rc=$? >> gpurun_out/r2c/tests.txt
tail -3 gpurun_out/r2c/tests.txt
for wl in "c2 --f2t-mode materialize" "c3 --f2t-mode materialize" "c4" "c2 --tensors yuv --f2t-mode materialize" "c4 --tensors yuv" "c3 --f2t-mode store" "c1"; do
  tag=$(echo $wl | tr ' -' '__')
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:f2t --csv --log-file gpurun_out/r2c/k_$tag.csv python bench.py --workload $wl --steps 1 --warmup 1 --frames 64 --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > /dev/null 2>&1
  echo "$wl: $(grep -o '"[^"]*f2t[^"]*"' gpurun_out/r2c/k_$tag.csv | sort | uniq -c | tr '\n' ' ')"
done

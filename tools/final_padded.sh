# round-2 final evidence with the scene-padded store: GPU suite, default bench, launch list, one strip capture
mkdir -p gpurun_out/fp
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/fp/gputests.log 2>&1; echo rc=$? >> gpurun_out/fp/gputests.log
tail -2 gpurun_out/fp/gputests.log
timeout -s KILL 600 python bench.py > gpurun_out/fp/bench.json 2> gpurun_out/fp/bench.err; python tools/show_bench.py gpurun_out/fp/bench.json
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config '' --no-compare-modes"
eval timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k "'regex:f2t|t2f|sad|cut_kernel'" --log-file gpurun_out/fp/launches_padded.csv $B > gpurun_out/fp/ncu_launch.log 2>&1
wc -l gpurun_out/fp/launches_padded.csv
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:f2t_strip420 --launch-skip 8 --launch-count 1 \
    -o gpurun_out/fp/r02d_c5padded_strip_full python bench.py --workload c5 --frames 1024 --steps 1 --warmup 1 --no-e2e \
    --no-cpu-baseline --per-config "" --no-compare-modes > gpurun_out/fp/ncu_full.log 2>&1
ls -la gpurun_out/fp/

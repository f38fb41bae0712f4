mkdir -p gpurun_out/prof3
C5="python bench.py --frames 256 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config '' --no-compare-modes --f2t-mode store"
eval $C5 > gpurun_out/prof3/plain.json 2>&1 || exit 1
eval ncu --set full --clock-control none --import-source on -k regex:f2t_strip -s 2 -c 1 -o gpurun_out/prof3/new_c5store_strip $C5 > gpurun_out/prof3/n1.log 2>&1
eval NNVISR_LIBNAME=libnnvisr_old.so ncu --set full --clock-control none --import-source on -k regex:f2t_strip -s 2 -c 1 -o gpurun_out/prof3/old_c5store_strip $C5 > gpurun_out/prof3/n2.log 2>&1
ls -la gpurun_out/prof3

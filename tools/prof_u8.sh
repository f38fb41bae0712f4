# ncu --set full of one c4 Fig. 1 batch launch (8-bit 720p strip kernel): current vs pre-rewrite build
mkdir -p gpurun_out/u8
for lib in libnnvisr.so libnnvisr_prev.so; do
 NNVISR_LIBNAME=$lib timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:f2t --launch-skip 3 --launch-count 1 \
   -o gpurun_out/u8/c4batch_${lib%.so} python bench.py --workload c4 --f2t-mode batch --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-config "" --no-compare-modes > gpurun_out/u8/${lib%.so}.log 2>&1
done
ls -la gpurun_out/u8

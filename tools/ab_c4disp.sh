# c4 (720p 8-bit) Fig. 1 batch slots (fan-out 1): strip kernel vs the TMA pipeline (NARROW two-CTA shape)
out=gpurun_out/ab_c4disp; mkdir -p $out
for rep in 1 2; do
 for s in 1 0; do
  NNVISR_F2T_STRIP=$s python bench.py --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes --workload c4 --f2t-mode batch > $out/c4batch_strip$s\_$rep.json 2>&1
 done
done
python tools/show_ab.py $out | sort

# c4 materialised (720p 8-bit, 2-frame windows: the NARROW two-CTA f2t_tma shape) launch knobs
out=gpurun_out/sweep_c4n; mkdir -p $out
B="python bench.py --workload c4 --per-config '' --no-e2e --no-cpu-baseline --no-compare-modes --steps 6"
for cfg in "base:" "b1:NNVISR_F2T_BAND=1" "b2:NNVISR_F2T_BAND=2" "b4:NNVISR_F2T_BAND=4" "s3:NNVISR_F2T_STAGES=3" \
           "s4:NNVISR_F2T_STAGES=4" "nob3:NNVISR_F2T_NOB=3" "st1:NNVISR_F2T_STORERS=1" "rf0:NNVISR_F2T_RELFIRST=0" \
           "b2s3:NNVISR_F2T_BAND=2 NNVISR_F2T_STAGES=3" "b1s3:NNVISR_F2T_BAND=1 NNVISR_F2T_STAGES=3" \
           "b1s4nob3:NNVISR_F2T_BAND=1 NNVISR_F2T_STAGES=4 NNVISR_F2T_NOB=3" "ct256:NNVISR_F2T_CT=256"; do
  name=${cfg%%:*}; env=${cfg#*:}
  for rep in 1 2; do eval env $env $B > $out/${name}_$rep.json 2>&1; done
done
python tools/show_ab.py $out | sort

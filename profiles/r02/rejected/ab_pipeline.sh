# pipelined directions (bench --pipeline: t2f on a second stream gated on f2t
# events) vs serial, with per-SM CTA caps that leave room for co-residency
out=gpurun_out/ab_pipeline; mkdir -p $out
B="python bench.py --per-config '' --no-e2e --no-cpu-baseline --no-compare-modes"
for rep in 1 2; do
 for v in base pipe pipe_t2 pipe_t2s1 pipe_t1s1; do
  case $v in
   base) E=""; P="";;
   pipe) E=""; P="--pipeline";;
   pipe_t2) E="NNVISR_T2F_MAXCTAS=2"; P="--pipeline";;
   pipe_t2s1) E="NNVISR_T2F_MAXCTAS=2 NNVISR_F2T_STRIP_MAXCTAS=1"; P="--pipeline";;
   pipe_t1s1) E="NNVISR_T2F_MAXCTAS=1 NNVISR_F2T_STRIP_MAXCTAS=1"; P="--pipeline";;
  esac
  eval env $E $B --workload c5 --frames 1024 $P > $out/c5_${v}_$rep.json 2>&1
  eval env $E $B --workload c2 $P > $out/c2_${v}_$rep.json 2>&1
 done
done
python tools/show_ab.py $out | sort

# same-box A/B of launch-size knobs on the default workload (c5, 1024 frames) and c2:
# t2f tuples per launch and strip tiles per resident CTA
out=gpurun_out/ab_knobs; mkdir -p $out
B="python bench.py --per-config '' --no-e2e --no-cpu-baseline --no-compare-modes"
for rep in 1 2; do
 for v in base t104 tpc28 tpc16; do
  case $v in
   base) E=""; P="";;
   t104) E=""; P="--t2f-chunk 104";;
   tpc28) E="NNVISR_F2T_STRIP_TPC=28"; P="";;
   tpc16) E="NNVISR_F2T_STRIP_TPC=16"; P="";;
  esac
  eval env $E $B --workload c5 --frames 1024 $P > $out/c5_${v}_$rep.json 2>&1
  eval env $E $B --workload c2 $P > $out/c2_${v}_$rep.json 2>&1
 done
done
python tools/show_ab.py $out | sort

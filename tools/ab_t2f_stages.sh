out=gpurun_out/${1:-abst}; mkdir -p $out
for rep in 1 2; do for st in 2 3; do
 NNVISR_T2F_STAGES=$st python bench.py --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/c5_st${st}_$rep.json 2>&1
done; done

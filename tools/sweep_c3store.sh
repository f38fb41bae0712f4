# f2t_tma knobs for c3 store mode (4:4:4 16-bit -> fp32, one slot per frame)
out=gpurun_out/${1:-swc3}; mkdir -p $out
run() { tag=$1; shift; env "$@" python bench.py --workload c3 --f2t-mode store --frames 240 --per-config "" --no-e2e --no-cpu-baseline --no-compare-modes > $out/$tag.json 2>&1; }
run base
run band1 NNVISR_F2T_BAND=1
run band4 NNVISR_F2T_BAND=4
run nob2 NNVISR_F2T_NOB=2
run nob4 NNVISR_F2T_NOB=4
run st3 NNVISR_F2T_STAGES=3
run loader0 NNVISR_F2T_LOADER=0
run base2

for lib in libnnvisr_e.so libnnvisr_b.so libnnvisr_e.so libnnvisr_b.so; do
 for spec in "c2 materialize" "c2 store" "c5 materialize" "c4 materialize" "c4 batch"; do set -- $spec
  NNVISR_LIBNAME=$lib python bench.py --workload $1 --frames 240 --f2t-mode $2 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/x.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/x.json'));v=d['per_direction']['f2t']; print('$lib $1 $2', round(v['achieved_gbs']), round(v['fps']))"
 done
done

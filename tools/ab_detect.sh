for r in 1 2; do for lib in libnnvisr_e.so libnnvisr_b.so; do for wl in c2 c4 c5; do NNVISR_LIBNAME=$lib python bench.py --workload $wl --detect --frames 240 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/x.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/x.json'));v=d['per_direction']['detect']; print('$lib $wl', round(v['achieved_gbs']), round(v['avg_launch_ms'],3))"; done; done; done
timeout 300 python -m pytest tests/test_gpu_scene.py -q -x 2>&1 | tail -1

# strip kernel tile queue (mbarrier slots, no CTA barrier per tile) vs the
# per-tile __syncthreads build (libnnvisr_old.so): tests, then same-box A/B
mkdir -p gpurun_out/tq
timeout -s KILL 300 python -m pytest tests/test_gpu_strip.py tests/test_gpu_store_ring.py tests/test_gpu_batch_store.py -q -x > gpurun_out/tq/tests.txt 2>&1; echo rc=$? >> gpurun_out/tq/tests.txt
tail -3 gpurun_out/tq/tests.txt
grep -q "rc=0" gpurun_out/tq/tests.txt || exit 1
LIBS="libnnvisr.so libnnvisr_old.so" timeout -s KILL 1200 bash tools/ab_lib.sh tq
python tools/show_ab.py gpurun_out/tq | sort
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/tq/gputests.log 2>&1; echo rc=$? >> gpurun_out/tq/gputests.log
tail -2 gpurun_out/tq/gputests.log

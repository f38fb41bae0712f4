mkdir -p gpurun_out/final3
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/final3/gputests.log 2>&1; echo rc=$? >> gpurun_out/final3/gputests.log
tail -2 gpurun_out/final3/gputests.log
timeout -s KILL 900 bash tools/checked_tests.sh > gpurun_out/final3/checked.log 2>&1; echo rc=$? >> gpurun_out/final3/checked.log
tail -2 gpurun_out/final3/checked.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3/smoke.log 2>&1; tail -1 gpurun_out/final3/smoke.log
timeout -s KILL 600 python bench.py > gpurun_out/final3/bench.json 2> gpurun_out/final3/bench.err; python tools/show_bench.py gpurun_out/final3/bench.json

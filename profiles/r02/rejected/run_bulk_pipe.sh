LIBS="libnnvisr.so libnnvisr_stg.so" bash tools/ab_lib.sh ab_bulk
python tools/show_ab.py gpurun_out/ab_bulk | sort
bash tools/ab_pipeline.sh

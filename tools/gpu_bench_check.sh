timeout 900 python bench.py --no-cpu-one-core > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 600 python tools/time_runs.py --config 4 --runs 6 > gpurun_out/time5_cfg4.txt 2>&1

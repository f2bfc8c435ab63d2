for c in 4 5 3 2; do timeout 600 python tools/time_runs.py --config $c --runs 4 > gpurun_out/time4_cfg$c.txt 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_configs.py tests/test_gpu_edge_cases.py tests/test_gpu_stages.py -q -x > gpurun_out/t_engine.log 2>&1; echo rc=$? >> gpurun_out/t_engine.log

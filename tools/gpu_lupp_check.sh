set -x
timeout 600 python -m pytest tests/test_gpu_stages.py -q -x -k lupp > gpurun_out/t_lupp.log 2>&1; echo rc=$? >> gpurun_out/t_lupp.log
for a in "100000 50 3" "100000 50 4" "100000 50 0" "50000 32 2" "50000 32 4" "50000 64 3" "50000 64 4" "60000 12 4" "200000 64 0" "20000 20 1" "20000 20 4"; do timeout 120 python tools/time_stage.py lupp $a 20; done > gpurun_out/lupp_times.txt 2>&1
for c in 4 3; do timeout 600 python tools/time_runs.py --config $c --runs 5 > gpurun_out/time2_cfg$c.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_configs.py tests/test_gpu_edge_cases.py -q -x > gpurun_out/t_engine.log 2>&1; echo rc=$? >> gpurun_out/t_engine.log

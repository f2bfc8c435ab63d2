timeout 600 python -m pytest tests/test_gpu_stages.py -q -x -k "rows_lu_solve" > gpurun_out/t_solve.log 2>&1; echo rc=$? >> gpurun_out/t_solve.log
for c in 4 5; do timeout 600 python tools/time_runs.py --config $c --runs 4 > gpurun_out/time6_cfg$c.txt 2>&1; ITERCUR_ROWS_SOLVE_BLK=1 timeout 600 python tools/time_runs.py --config $c --runs 3 > gpurun_out/time6_blk_cfg$c.txt 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:rows_lu_solve --log-file gpurun_out/launches_solve.csv python tools/profile_run.py --config 4 --runs 1 > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_configs.py tests/test_gpu_edge_cases.py -q -x > gpurun_out/t_engine.log 2>&1; echo rc=$? >> gpurun_out/t_engine.log

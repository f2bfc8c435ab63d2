# launch list of one config-4 run (second run in the process) + phase timings
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv \
    python tools/profile_run.py --config 4 --runs 2 > gpurun_out/ncu_launch_cfg4.log 2>&1
timeout 600 python tools/ab_phases.py --help > gpurun_out/ab_help.txt 2>&1

#!/bin/bash
# Diagnose config-5 time (phases, host trace) and the config-4 host gaps.
nvidia-smi --query-gpu=name,power.limit,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/diag_smi.txt 2>&1
python tools/ab_phases.py 5 3 '' > gpurun_out/diag_phases_cfg5.txt 2>&1
python tools/ab_phases.py 4 3 '' > gpurun_out/diag_phases_cfg4.txt 2>&1
ITERCUR_HOST_TRACE=1 python tools/time_runs.py --config 5 --runs 4 > gpurun_out/diag_trace_cfg5.txt 2>&1
ITERCUR_HOST_TRACE=1 python tools/time_runs.py --config 4 --runs 4 > gpurun_out/diag_trace_cfg4.txt 2>&1
ITERCUR_HOST_TRACE=1 python tools/time_runs.py --config 2 --runs 3 > gpurun_out/diag_trace_cfg2.txt 2>&1

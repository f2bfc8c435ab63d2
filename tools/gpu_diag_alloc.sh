#!/bin/bash
ITERCUR_HOST_TRACE=1 timeout 600 python tools/time_runs.py --config 2 --runs 14 > gpurun_out/alloc_trace_cfg2.txt 2>&1
timeout 600 python tools/time_runs.py --config 5 --runs 8 > gpurun_out/time_r02h_cfg5.txt 2>&1

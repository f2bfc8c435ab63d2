#!/bin/bash
# After moving every allocation of a run ahead of the sketch enqueue (big buffers first).
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02g.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r02g.log
ITERCUR_HOST_TRACE=1 timeout 600 python tools/time_runs.py --config 2 --runs 14 > gpurun_out/time_r02g_cfg2.txt 2>&1
ITERCUR_HOST_TRACE=1 timeout 600 python tools/time_runs.py --config 4 --runs 14 > gpurun_out/time_r02g_cfg4.txt 2>&1
for c in 1 3 5; do timeout 600 python tools/time_runs.py --config $c --runs 8 > gpurun_out/time_r02g_cfg$c.txt 2>&1; done
timeout 1500 python bench.py > gpurun_out/bench_r02g.json 2> gpurun_out/bench_r02g.err

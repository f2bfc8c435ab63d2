#!/bin/bash
# After deferring the sketch's host sync behind the first batch's graph capture/upload.
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02f.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r02f.log
for c in 4 2 5 3 1; do ITERCUR_HOST_TRACE=1 timeout 600 python tools/time_runs.py --config $c --runs 6 > gpurun_out/time_r02f_cfg$c.txt 2>&1; done

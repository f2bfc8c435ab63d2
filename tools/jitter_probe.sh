#!/bin/bash
# Does the run-to-run allocation jitter (GB-sized pool requests taking ms) depend on what ran on
# the box before? Device times of config 2 on a quiet box, then after the GPU suite.
probe() {
  echo "== $1"; nvidia-smi --query-compute-apps=pid,used_memory --format=csv; nvidia-smi --query-gpu=memory.used,memory.total --format=csv
  free -g | head -2; grep -E "AnonHugePages|HugePages_Total|MemAvailable" /proc/meminfo
}
probe "quiet box" > gpurun_out/jitter_env.txt 2>&1
ITERCUR_HOST_TRACE=1 timeout 600 python tools/time_runs.py --config 2 --runs 14 > gpurun_out/jitter_quiet_cfg2.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/jitter_pytest.log 2>&1
probe "after the GPU suite" >> gpurun_out/jitter_env.txt 2>&1
ITERCUR_HOST_TRACE=1 timeout 600 python tools/time_runs.py --config 2 --runs 14 > gpurun_out/jitter_after_cfg2.txt 2>&1
probe "end" >> gpurun_out/jitter_env.txt 2>&1

#!/bin/bash
# GPU-box check of the current tree: the GPU suite, smoke, and per-config device times.
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for c in 1 2 3 4 5; do timeout 600 python tools/time_runs.py --config $c --runs 4 > gpurun_out/time_cfg$c.txt 2>&1; done

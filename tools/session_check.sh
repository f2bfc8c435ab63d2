#!/bin/bash
# GPU-box check of the current tree: GPU suite, smoke, per-config timings (profile mode), bench line.
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for c in 2 4; do timeout 600 python tools/time_runs.py --config $c --runs 5 --profile-first > gpurun_out/time_cfg$c.txt 2>&1; done
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err

#!/bin/bash
# Re-entry check of the rebuilt tree: GPU suite, smoke, both bench arms, per-config device times.
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02e.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r02e.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02e.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_r02e.json 2> gpurun_out/bench_r02e.err
timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref_r02e.json 2> gpurun_out/bench_ref_r02e.err
for c in 1 2 3 4 5; do timeout 600 python tools/time_runs.py --config $c --runs 5 > gpurun_out/time_r02e_cfg$c.txt 2>&1; done

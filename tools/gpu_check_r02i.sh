#!/bin/bash
# Round-2 closing check at the final commit: GPU suite, smoke, both bench arms, device times.
timeout 1500 python bench.py > gpurun_out/bench_r02i.json 2> gpurun_out/bench_r02i.err
timeout 1500 python bench.py --impl reference --steps 5 > gpurun_out/bench_ref_r02i.json 2> gpurun_out/bench_ref_r02i.err
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02i.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r02i.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02i.log 2>&1
for c in 1 2 3 4 5; do timeout 600 python tools/time_runs.py --config $c --runs 8 > gpurun_out/time_r02i_cfg$c.txt 2>&1; done

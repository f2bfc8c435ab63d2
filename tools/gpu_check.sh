#!/bin/bash
# GPU-box check of the current tree (round-2 closing run: profiles/bench_r02_final_cfg4.json, gputest_r02_final.txt,
# time_runs_r02_final.txt): both bench arms, the GPU suite, smoke, device times of the five configs. ITERCUR_HOST_TRACE=1
# in front of tools/time_runs.py prints the host timeline of every run (set-up marks, allocations, batches).
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 1500 python bench.py --impl reference --steps 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for c in 1 2 3 4 5; do timeout 600 python tools/time_runs.py --config $c --runs 8 > gpurun_out/time_cfg$c.txt 2>&1; done

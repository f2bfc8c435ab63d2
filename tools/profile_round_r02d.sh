#!/bin/bash
# Round-2 closing profile (after tools/profile_round_r02c.sh's parity run; later changes keep the
# arithmetic): bench line (config 4) and reference arm, launch lists of config 2/4/5 runs, ncu
# --set full captures of the per-iteration kernels in a config-4 run, the GPU suite, device times.
set -x
timeout 1500 python bench.py > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err
timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref_r02d.json 2> gpurun_out/bench_ref_r02d.err
for c in 2 4 5; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02d_cfg$c.csv \
      python tools/profile_run.py --config $c --runs 1 > gpurun_out/ncu_launch_r02d_cfg$c.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"lupp_resident|ts_gemm_lean|rows_lu_solve_mma" -s 10 -c 6 \
    -o gpurun_out/full_r02d_cfg4_iter python tools/profile_run.py --config 4 --runs 1 > gpurun_out/ncu_full_iter_d.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r02d.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02d.log 2>&1
for c in 1 2 3 4 5; do timeout 600 python tools/time_runs.py --config $c --runs 5 > gpurun_out/time_r02d_cfg$c.txt 2>&1; done

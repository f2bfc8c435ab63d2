#!/bin/bash
# Round-2 (second session) profile: bench line (config 4), reference arm, launch list of one
# config-4 run, ncu --set full captures of the resident LUPP and the lean GEMMs in a config-4 run.
set -x
timeout 1500 python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err
timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref_r02b.json 2> gpurun_out/bench_ref_r02b.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02b_cfg4.csv \
    python tools/profile_run.py --config 4 --runs 1 > gpurun_out/ncu_launch_r02b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"lupp_resident" -s 2 -c 1 \
    -o gpurun_out/full_r02b_cfg4_lupp python tools/profile_run.py --config 4 --runs 1 > gpurun_out/ncu_full_lupp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ts_gemm_lean" -s 6 -c 3 \
    -o gpurun_out/full_r02b_cfg4_gemm python tools/profile_run.py --config 4 --runs 1 > gpurun_out/ncu_full_gemm.log 2>&1

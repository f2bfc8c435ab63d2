#!/bin/bash
# Round-2 closing profile at the final engine (sketch read-back deferred behind the first batch's
# graph capture): bench line (config 4) and reference arm, launch lists of config 2/4/5 runs,
# ncu --set full of the sketch and per-iteration kernels at config 4 (summarised on the box: the
# reports with sources exceed what gpurun copies back), device times of all configs.
set -x
timeout 1500 python bench.py > gpurun_out/bench_r02f.json 2> gpurun_out/bench_r02f.err
timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref_r02f.json 2> gpurun_out/bench_ref_r02f.err
for c in 2 4 5; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02f_cfg$c.csv \
      python tools/profile_run.py --config $c --runs 1 > gpurun_out/ncu_launch_r02f_cfg$c.log 2>&1
done
mkdir -p /tmp/ncu_f
ncu --set full --clock-control none --import-source on -k regex:"sparse_sketch_umma|lupp_resident|ts_gemm_lean|rows_lu_solve_mma" -c 8 \
    -f -o /tmp/ncu_f/full_r02f_cfg4 python tools/profile_run.py --config 4 --runs 1 > gpurun_out/ncu_full_f.log 2>&1
python tools/summarize_ncu.py full /tmp/ncu_f/full_r02f_cfg4.ncu-rep > gpurun_out/ncu_full_r02f_cfg4.txt 2> gpurun_out/ncu_full_r02f_cfg4.err
for c in 1 3 4 5; do timeout 600 python tools/time_runs.py --config $c --runs 6 > gpurun_out/time_r02f2_cfg$c.txt 2>&1; done
ITERCUR_HOST_TRACE=1 timeout 600 python tools/time_runs.py --config 2 --runs 12 > gpurun_out/time_r02f2_cfg2.txt 2>&1
du -sh gpurun_out

#!/bin/bash
# Round-2 profile on the GPU box: bench line (config 4, no profiler), the reference arm, the ncu
# launch list of one config-4 run, and `--set full` captures of the sketch kernel at configs 3/4/5.
# Outputs in gpurun_out/ (summaries go to profiles/ via tools/summarize_ncu.py).
set -x
timeout 1500 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref_r02.json 2> gpurun_out/bench_ref_r02.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_cfg4.csv \
    python tools/profile_run.py --config 4 --runs 1 > gpurun_out/ncu_launch_cfg4.log 2>&1
for c in 4 3 5; do
  ncu --set full --clock-control none --import-source on -k regex:"sparse_sketch_imma|sparse_sketch_umma|sketch_dmma" -c 1 \
      -o gpurun_out/full_r02_cfg${c}_sketch python tools/profile_run.py --config $c --sketch-only --runs 1 \
      > gpurun_out/ncu_full_cfg${c}.log 2>&1
done

# Round profile: GPU tests, smoke, bench line (no profiler), the ncu launch list of one config-2
# run, and `--set full` captures of the sketch kernel and the per-iteration kernels. Outputs in gpurun_out/.
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v6.csv \
    python tools/profile_run.py --config 2 --runs 1 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sparse_sketch_imma|sparse_sketch_umma|sketch_dmma" -c 1 \
    -o gpurun_out/full_v6_sketch python tools/profile_run.py --config 2 --runs 1 > gpurun_out/ncu_full1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"lupp_cluster_v2|ts_gemm_lean|gather_pair" -s 200 -c 5 \
    -o gpurun_out/full_v6_iter python tools/profile_run.py --config 2 --runs 1 > gpurun_out/ncu_full2.log 2>&1

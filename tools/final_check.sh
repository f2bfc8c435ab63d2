# Full GPU tests, smoke, config sweep 1-5 (warm, true errors), bench line.
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1800 python tools/config_sweep.py --true-error > gpurun_out/config_sweep.jsonl 2> gpurun_out/config_sweep.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err

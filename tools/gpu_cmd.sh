timeout 600 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_sharded.log 2>&1
timeout 900 python bench.py --sharded --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_sharded_sketch.json 2>gpurun_out/bench_sharded.err

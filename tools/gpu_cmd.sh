timeout 900 python -m pytest tests/test_gpu_engine.py -x -q -k "matches_oracle" > gpurun_out/pytest_engine.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_engine.log

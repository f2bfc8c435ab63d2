python -m pytest tests/test_gpu_stages.py -x -q -k "sparse or sketch" > gpurun_out/pytest_stages.log 2>&1
for ns in 6 7; do ITERCUR_IMMA_SLICES=$ns python tools/sketch_modes.py 20000 10000 20 40000 20000 50 100000 50000 50 2>&1 | grep '"2"' | sed "s/^/ns=$ns /"; done > gpurun_out/sketch_ns.txt

export ITERCUR_SPARSE_SKETCH=2
ncu --set full --clock-control none --import-source on -k regex:sparse_sketch_imma -s 1 -c 1 -o gpurun_out/imma_full python tools/sketch_one.py 40000 20000 50 sparse_sign 2 > gpurun_out/ncu_imma.log 2>&1
python -m pytest tests/test_gpu_stages.py -x -q -k "sparse or sketch" > gpurun_out/pytest_stages.log 2>&1

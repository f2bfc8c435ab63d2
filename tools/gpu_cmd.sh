timeout 1500 python tools/config_sweep.py --true-error > gpurun_out/config_sweep.jsonl 2> gpurun_out/config_sweep.err
ncu --set full --clock-control none --import-source on -k regex:sparse_sketch_umma -c 1 -o gpurun_out/full_v5_umma python tools/sketch_one.py 100000 50000 50 sparse_sign 1 > gpurun_out/ncu_umma.log 2>&1

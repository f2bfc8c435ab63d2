ncu --set full --clock-control none --import-source on -k regex:lupp_resident -c 1 -o gpurun_out/res_small python tools/time_stage.py lupp 4736 50 4 2 > gpurun_out/res_ncu_small.log 2>&1

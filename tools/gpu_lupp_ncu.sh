ncu --set full --clock-control none --import-source on -k regex:lupp_resident -c 1 -o gpurun_out/res_full50 python tools/time_stage.py lupp 100000 50 4 2 > gpurun_out/res_ncu50.log 2>&1

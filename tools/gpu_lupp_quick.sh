timeout 600 python -m pytest tests/test_gpu_stages.py -q -x -k lupp > gpurun_out/t_lupp.log 2>&1; echo rc=$? >> gpurun_out/t_lupp.log
for a in "100000 50 4" "50000 32 4" "50000 64 4" "4736 50 4"; do timeout 120 python tools/time_stage.py lupp $a 20; done > gpurun_out/lupp_times.txt 2>&1
for a in "4736 50 4" "100000 50 4"; do ITERCUR_LIB_OVERRIDE=tools/altlibs/restrace.so ITERCUR_LUPP_TRACE=1 timeout 120 python tools/time_stage.py lupp $a 3; done > gpurun_out/lupp_trace.txt 2>&1
for a in "4736 50 4" "100000 50 4"; do echo "== $a"; ITERCUR_LIB_OVERRIDE=tools/altlibs/restrace.so ITERCUR_LUPP_GTRACE=1 timeout 120 python tools/time_stage.py lupp $a 3; done > gpurun_out/lupp_gtrace.txt 2>&1

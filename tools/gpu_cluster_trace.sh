for a in "10000 20 1" "20000 20 1"; do ITERCUR_LIB_OVERRIDE=tools/altlibs/instr.so ITERCUR_LUPP_TRACE=1 timeout 120 python tools/time_stage.py lupp $a 5; done > gpurun_out/cluster_trace.txt 2>&1
for a in "10000 20 1" "20000 20 1" "10000 20 4" "20000 20 4"; do timeout 120 python tools/time_stage.py lupp $a 20; done > gpurun_out/cluster_times.txt 2>&1

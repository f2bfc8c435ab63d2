for a in "4736 50 4" "100000 50 4"; do ITERCUR_LIB_OVERRIDE=tools/altlibs/restrace.so ITERCUR_LUPP_TRACE=1 timeout 120 python tools/time_stage.py lupp $a 3; done > gpurun_out/lupp_trace.txt 2>&1

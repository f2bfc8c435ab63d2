for lib in "" tools/altlibs/ldcg.so tools/altlibs/ldvol.so; do
  echo "== lib ${lib:-default}"
  for a in "4736 12 4" "4736 50 4" "29600 50 4" "100000 50 4"; do ITERCUR_LIB_OVERRIDE=$lib timeout 120 python tools/time_stage.py lupp $a 20; done
done > gpurun_out/lupp_ab.txt 2>&1
ITERCUR_LUPP_TRACE=1 timeout 120 python tools/time_stage.py lupp 4736 50 4 5 > gpurun_out/lupp_trace_small.txt 2>&1

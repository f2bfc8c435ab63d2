for a in "4736 50 4" "100000 50 4"; do echo "== $a"; ITERCUR_LUPP_GTRACE=1 timeout 120 python tools/time_stage.py lupp $a 3; done > gpurun_out/lupp_gtrace.txt 2>&1

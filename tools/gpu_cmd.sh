ITERCUR_HOST_TRACE=1 python tools/time_runs.py --config 2 --runs 30 > gpurun_out/tr_trace.txt 2> gpurun_out/tr_trace.err

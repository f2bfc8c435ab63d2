for i in 1 2; do
python tools/time_runs.py --config 2 --runs 8 > gpurun_out/tr_pair_$i.txt 2>&1
ITERCUR_NO_PAIR_GATHER=1 python tools/time_runs.py --config 2 --runs 8 > gpurun_out/tr_nopair_$i.txt 2>&1
done

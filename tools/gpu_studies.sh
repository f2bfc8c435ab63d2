#!/bin/bash
# The round-2 kernel studies behind DESIGN.md §4 (run on the GPU box with gpurun; outputs in
# gpurun_out/). Pick one with the first argument.
#   lupp    resident vs panel vs cluster LUPP timings at the config shapes, and the resident kernel's
#           per-step traces (CTA-0 phases with ITERCUR_LUPP_TRACE, every CTA's exchange skew with
#           ITERCUR_LUPP_GTRACE; both need the trace build: python tools/build_variant.py restrace
#           -DITERCUR_RES_TRACE)
#   exchange the pure exchange floor (tools/microbench/res_exchange.cu) and warp-reduction latency
#   gemm    lean/generic x base-in-shared-memory sweep at the config 4/5 GEMM shapes
#   roles   per-role times of the three per-iteration GEMMs in config 4/5 runs (tools/gemm_roles.py)
#   solve   the row solves: tensor-core vs scalar blocked form (parity test + config 4/5 run times)
#   sketch  tcgen05 vs mma.sync sparse-sign sketch at config 2
case "$1" in
  lupp)
    for a in "100000 50 4" "100000 50 3" "50000 32 4" "50000 32 2" "50000 64 4" "60000 12 4" "200000 64 0" \
             "10000 20 1" "20000 20 1" "20000 20 4"; do timeout 120 python tools/time_stage.py lupp $a 20; done \
      > gpurun_out/lupp_times.txt 2>&1
    for a in "4736 50 4" "100000 50 4"; do
      ITERCUR_LIB_OVERRIDE=tools/altlibs/restrace.so ITERCUR_LUPP_TRACE=1 timeout 120 python tools/time_stage.py lupp $a 3
      ITERCUR_LIB_OVERRIDE=tools/altlibs/restrace.so ITERCUR_LUPP_GTRACE=1 timeout 120 python tools/time_stage.py lupp $a 3
    done > gpurun_out/lupp_traces.txt 2>&1 ;;
  exchange)
    (timeout 120 tools/microbench/res_exchange; timeout 60 tools/microbench/warp_lat) > gpurun_out/exchange_floor.txt 2>&1 ;;
  gemm)
    for shape in "100000 50" "200000 64" "50000 64" "100000 56"; do for K in 64 256 512 1024; do
      for v in "4 0" "4 1" "5 0" "5 1" "6 1" "-1 0"; do set -- $v
        ITERCUR_GEMM_LEAN=$1 ITERCUR_GEMM_BSM=$2 timeout 60 python tools/time_stage.py gemm $shape $K 10 | sed "s/^/lean=$1 bsm=$2 /"
      done; done; done > gpurun_out/gemm_sweep.txt 2>&1 ;;
  roles)
    for c in 4 5; do
      ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/roles_cfg$c.csv \
          python tools/profile_run.py --config $c --runs 1 > /dev/null 2>&1
      python tools/gemm_roles.py gpurun_out/roles_cfg$c.csv > gpurun_out/roles_cfg$c.txt
    done ;;
  solve)
    timeout 600 python -m pytest tests/test_gpu_stages.py -q -x -k rows_lu_solve > gpurun_out/solve_tests.log 2>&1
    for c in 4 5; do for blk in 0 1; do echo "config $c ITERCUR_ROWS_SOLVE_BLK=$blk"
      ITERCUR_ROWS_SOLVE_BLK=$blk timeout 600 python tools/time_runs.py --config $c --runs 4 2>&1 | tail -2; done; done \
      > gpurun_out/solve_ab.txt 2>&1 ;;
  sketch)
    for m in 2 3; do echo "ITERCUR_SPARSE_SKETCH=$m"
      ITERCUR_SPARSE_SKETCH=$m timeout 300 python tools/time_stage.py sketch 20000 10000 20 sparse_sign 20
      ITERCUR_SPARSE_SKETCH=$m timeout 600 python tools/time_runs.py --config 2 --runs 4 2>&1 | tail -2; done \
      > gpurun_out/sketch_ab.txt 2>&1 ;;
  *) echo "usage: tools/gpu_studies.sh lupp|exchange|gemm|roles|solve|sketch"; exit 1 ;;
esac

# generic tall-skinny GEMM at the config-4/5 shapes: warps per CTA and split-K (tools/time_stage.py gemm)
for W in 2 4 8; do
  for K in 100 200 400; do
    echo -n "warps=$W M=100000 N=50 K=$K: "; ITERCUR_GEMM_WARPS=$W python tools/time_stage.py gemm 100000 50 $K 20
  done
  for K in 256 1024; do echo -n "warps=$W M=200000 N=64 K=$K: "; ITERCUR_GEMM_WARPS=$W python tools/time_stage.py gemm 200000 64 $K 10; done
done
for S in 2 4; do for K in 200 400; do echo -n "splits=$S M=100000 N=50 K=$K: "; ITERCUR_GEMM_SPLITS=$S python tools/time_stage.py gemm 100000 50 $K 20; done; done

for L in -1 1 2 3; do
  for K in 100 200 400; do
    echo -n "lean=$L K=$K: "; ITERCUR_GEMM_LEAN=$L python tools/time_stage.py gemm 100000 50 $K 20
  done
done
for L in -1 2; do for K in 256 512 1024; do echo -n "lean=$L M=200000 N=64 K=$K: "; ITERCUR_GEMM_LEAN=$L python tools/time_stage.py gemm 200000 64 $K 10; done; done

"""Tall-skinny GEMM timing vs the HBM / FP64 bounds, for the per-iteration shapes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_21963_b200 import stages
for M, N, K in ((20000, 20, 1200), (20000, 20, 2400), (10000, 20, 1200), (10000, 20, 2400), (200000, 64, 512),
                (50000, 64, 512), (50000, 32, 128), (100000, 50, 200)):
    us = stages.time_gemm(M, N, K, reps=10)
    byts = 8.0 * M * K
    fl = 2.0 * M * ((N + 7) // 8 * 8) * K
    print(json.dumps({"M": M, "N": N, "K": K, "us": round(us, 1), "hbm_us": round(byts / 6452e9 * 1e6, 1),
                      "fp64_us": round(fl / 37.1e12 * 1e6, 1),
                      "frac_of_bound": round(max(byts / 6452e9, fl / 37.1e12) * 1e6 / us, 3),
                      "warps_env": os.environ.get("ITERCUR_GEMM_WARPS", "auto")}), flush=True)

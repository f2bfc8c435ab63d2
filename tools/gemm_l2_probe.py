"""Row-residual GEMM (M x 20, K) time per byte of L as K grows past the L2 (126 MB):
does the kernel speed up when L is L2-resident?  python tools/gemm_l2_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_21963_b200 import stages  # noqa: E402

for K in (100, 200, 400, 600, 800, 1180, 1600, 2400):
    us = stages.time_gemm(20000, 20, K, reps=20)
    mb = 20000 * K * 8 / 1e6
    print(f"K={K:5d} L={mb:7.1f} MB  {us:8.2f} us  {mb * 1e6 / (us * 1e-6) / 1e9:8.1f} GB/s  "
          f"{2 * 20000 * 24 * K / (us * 1e-6) / 1e12:6.2f} TF/s(24-wide)", flush=True)

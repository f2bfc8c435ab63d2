"""Time one sketch apply on an m x n Gaussian matrix (ncu target):
    python tools/sketch_one.py M N B KIND [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_21963_b200 import stages  # noqa: E402

m, n, b, kind = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
a = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
print(m, n, b, kind, stages.time_sketch_kernel(a, b, kind=kind, reps=reps))

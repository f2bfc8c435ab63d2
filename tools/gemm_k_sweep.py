import sys, os
sys.path.insert(0, os.getcwd())
from paper_2509_21963_b200 import stages
for K in (1, 100, 200, 400, 800, 1600, 2400):
    print(os.environ.get("ITERCUR_GEMM_SPLITS", "auto"), K, round(stages.time_gemm(20000, 20, K, reps=20), 2), round(stages.time_gemm(10000, 20, K, reps=20), 2))

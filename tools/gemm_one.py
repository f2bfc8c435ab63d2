import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_21963_b200 import stages
M, N, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
print(stages.time_gemm(M, N, K, reps=2))

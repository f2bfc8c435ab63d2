import sys, os
sys.path.insert(0, os.getcwd())
from paper_2509_21963_b200 import stages
for rows, steps in [(200000, 64), (100000, 50), (200000, 32), (50000, 64)]:
    print(rows, steps, stages.time_lupp(rows, steps, reps=10))

import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_21963_b200 import stages
rows, steps, path = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
print(stages.time_lupp(rows, steps, reps=2, force_path=path))

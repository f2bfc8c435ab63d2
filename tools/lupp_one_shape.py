"""Time one LUPP shape (rows x steps) through stages.time_lupp; for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_21963_b200 import stages  # noqa: E402

rows, steps = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
print(rows, steps, stages.time_lupp(rows, steps, reps=reps))

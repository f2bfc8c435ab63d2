"""LUPP kernel latency: fixed cost vs per-step cost for each path (cluster / grid smem / global)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_21963_b200 import stages
for rows, steps_list in ((10000, (1, 2, 5, 10, 20)), (20000, (1, 5, 20)), (50000, (1, 32)), (100000, (1, 50)),
                         (200000, (1, 64))):
    for steps in steps_list:
        out = {"rows": rows, "steps": steps}
        for path, name in ((1, "cluster"), (2, "grid"), (3, "global")):
            try:
                r = stages.time_lupp(rows, steps, reps=20, force_path=path)
                out[name] = round(r["us"], 1)
                out[name + "_path"] = r["path"]
            except Exception as e:  # path not applicable
                out[name] = None
        print(json.dumps(out), flush=True)

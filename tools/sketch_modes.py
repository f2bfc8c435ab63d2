"""Sparse-sign sketch kernels side by side (ITERCUR_SPARSE_SKETCH = 0 dense DMMA, 1 list walk,
2 sliced-integer IMMA): ms per launch of the dominant kernel and the fraction of HBM peak.
    python tools/sketch_modes.py [M N B ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_21963_b200 import stages  # noqa: E402

HBM = 6452.2
shapes = [(20000, 10000, 20), (40000, 20000, 50), (100000, 50000, 50)]
if len(sys.argv) > 3:
    v = [int(x) for x in sys.argv[1:]]
    shapes = [tuple(v[i:i + 3]) for i in range(0, len(v), 3)]
for m, n, b in shapes:
    a = torch.empty(n, m, dtype=torch.float64, device="cuda").t()
    for j0 in range(0, n, 4096):  # fill in slabs (bounded temporary memory)
        a[:, j0:j0 + 4096].normal_()
    for mode in os.environ.get("SKETCH_MODES", "0,2,1").split(","):
        if mode == "1" and m * n > 1e9:
            continue
        os.environ["ITERCUR_SPARSE_SKETCH"] = mode
        r = stages.time_sketch_kernel(a, b, kind="sparse_sign", reps=5)
        gbs = 8.0 * m * n / (r["ms"] * 1e-3) / 1e9
        print(json.dumps({"m": m, "n": n, "b": b, "mode": mode, **r, "GBps": round(gbs, 1),
                          "frac_hbm": round(gbs / HBM, 3)}), flush=True)
    del a
    torch.cuda.empty_cache()

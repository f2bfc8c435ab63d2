"""A/B of per-phase device time (profile mode: CUDA events between the phases of every
iteration) under env switches: python tools/ab_phases.py CFG REPS 'ENV=1' '' ...
Each variant runs in its own process; prints the median over REPS of each phase sum (ms)."""
import json
import os
import subprocess
import sys

cfg, reps = sys.argv[1], int(sys.argv[2])
variants = sys.argv[3:]
code = r'''
import sys, json, torch
sys.path.insert(0, ".")
import paper_2509_21963_b200 as E
from paper_2509_21963_b200 import testmat
c = testmat.CONFIGS[int(sys.argv[1])]
a = testmat.generate(int(sys.argv[1])); torch.cuda.synchronize()
h = E.MatrixHandle.device(a)
kw = dict(epsilon=c["epsilon"], b=c["b"], seed=0, sketch=c["sketch"], max_rank=c["max_rank"])
out = []
for i in range(int(sys.argv[2]) + 1):
    f, t = E.iterative_cur(h, profile=True, **kw)
    ph = {k: sum(getattr(r, k) for r in t.iterations) * 1e3 for k in
          ("select_cols_s", "row_residual_s", "select_rows_s", "core_s", "downdate_s")}
    if i: out.append(ph)
    del f, t
print(json.dumps(out))
'''
for v in variants:
    env = dict(os.environ)
    for kv in v.split():
        k, val = kv.split("=", 1)
        env[k] = val
    r = subprocess.run([sys.executable, "-c", code, cfg, str(reps)], env=env, capture_output=True, text=True)
    if r.returncode:
        print(v, "FAILED", r.stderr[-500:])
        continue
    runs = json.loads(r.stdout.strip().splitlines()[-1])
    keys = runs[0].keys()
    med = {k: sorted(x[k] for x in runs)[len(runs) // 2] for k in keys}
    tot = sum(med.values())
    print(f"{v or '(default)':40s} total {tot:7.2f} ms  " + "  ".join(f"{k[:-2]} {med[k]:6.2f}" for k in keys))

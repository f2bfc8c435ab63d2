"""A/B timing of config runs under env switches: python tools/ab_runs.py CFG REPS 'ENV=1' '' ...
Each variant runs in its own process (switches are read once); variants alternate; min and
median of the device-timed runs after one warm-up are printed per variant."""
import json, os, subprocess, sys
cfg, reps = sys.argv[1], int(sys.argv[2])
variants = sys.argv[3:]
code = r'''
import sys, os, json, torch
sys.path.insert(0, ".")
import paper_2509_21963_b200 as E
from paper_2509_21963_b200 import testmat
c = testmat.CONFIGS[int(sys.argv[1])]
a = testmat.generate(int(sys.argv[1])); torch.cuda.synchronize()
h = E.MatrixHandle.device(a)
kw = dict(epsilon=c["epsilon"], b=c["b"], seed=0, sketch=c["sketch"], max_rank=c["max_rank"])
out = []
for i in range(int(sys.argv[2]) + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); f, t = E.iterative_cur(h, **kw); e1.record(); torch.cuda.synchronize()
    if i: out.append(e0.elapsed_time(e1))
    del f, t
print(json.dumps(out))
'''
res = {v: [] for v in variants}
for rnd in range(2):
    for v in variants:
        env = dict(os.environ)
        for kv in v.split():
            k, val = kv.split("=", 1)
            env[k] = val
        r = subprocess.run([sys.executable, "-c", code, cfg, str(reps)], env=env, capture_output=True, text=True)
        try:
            res[v] += json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            print(v, r.stderr[-500:])
for v, xs in res.items():
    xs = sorted(xs)
    print(f"{v or '(default)':40s} min {xs[0]:.2f} ms  median {xs[len(xs)//2]:.2f} ms  n={len(xs)}")

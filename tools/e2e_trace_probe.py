import sys, time, os
sys.path.insert(0, "/root/repo")
import torch
import paper_2509_21963_b200 as E
from paper_2509_21963_b200 import testmat
a = testmat.generate(4)
m, n = a.shape
host = torch.empty(n, m, dtype=torch.float64, pin_memory=True)
host.copy_(a.t()); del a; torch.cuda.empty_cache()
h = E.MatrixHandle.dense(host.numpy().T)
kw = dict(epsilon=1e-6, b=50, seed=0, sketch="sparse_sign")
for i in range(4):
    t0 = time.perf_counter(); f, t = E.iterative_cur(h, **kw); _ = f.row_indices; t1 = time.perf_counter()
    del f, t
    t2 = time.perf_counter()
    print(f"call {i}: {1e3*(t1-t0):.1f} ms (+ free {1e3*(t2-t1):.1f} ms)", file=sys.stderr, flush=True)

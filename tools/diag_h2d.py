import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np, ctypes as C
n = 200_000_000  # 1.6 GB
x = torch.empty(n, dtype=torch.float64, pin_memory=True)
x.fill_(1.0)
y = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize()
    print("torch pinned H2D GB/s", 1.6 / (time.perf_counter() - t0))
xp = torch.empty(n, dtype=torch.float64); xp.fill_(1.0)
torch.cuda.synchronize(); t0 = time.perf_counter(); y.copy_(xp); torch.cuda.synchronize()
print("torch pageable H2D GB/s", 1.6 / (time.perf_counter() - t0))
import paper_2509_21963_b200 as E
from paper_2509_21963_b200 import _capi
L = _capi.lib()
# time our host entry copy path only: a tiny run on a 20000 x 10000 pinned matrix with eps >= 1 (returns after sketch)
a = x[:200_000_000].view(10000, 20000).numpy().T  # (20000, 10000) F-order view of pinned memory
h = E.MatrixHandle.dense(a)
for _ in range(2):
    t0 = time.perf_counter(); f, t = E.iterative_cur(h, epsilon=2.0, b=20, sketch="sparse_sign"); dt = time.perf_counter() - t0
    print("host entry (copy + sketch) s", dt, "sketch_s", t.sketch_s, "total_s", t.total_s)

import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_21963_b200 as E
from oracle import oracle
m, n = 200000, 120
a = oracle.random_gaussian(m, 40, 5) @ oracle.random_gaussian(n, 40, 6).T
a += 1e-6 * oracle.random_gaussian(m, n, 7)
kw = dict(epsilon=1e-9, b=int(sys.argv[1]) if len(sys.argv) > 1 else 32, seed=1)
f, t = E.iterative_cur(a, **kw)
o = oracle.iterative_cur(a, **kw)
print("engine", t.status, f.rank, f.row_indices[:12])
print("oracle", o.status, len(o.row_indices), list(o.row_indices[:12]))
print("same I", f.row_indices == list(o.row_indices), "same J", f.col_indices == list(o.col_indices))
core = f.core_matrix()
X = a[np.ix_(f.row_indices, f.col_indices)]
print("core*X - I", np.linalg.norm(core @ X - np.eye(f.rank)))

import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from oracle import oracle as O
import paper_2509_21963_b200 as E
from parity_util import compare_runs
def lrn(m, n, r, rel, seed):
    a = O.random_gaussian(m, r, seed) @ O.random_gaussian(n, r, seed + 1).T
    noise = O.random_gaussian(m, n, seed + 2)
    return a + (rel * np.linalg.norm(a) / np.linalg.norm(noise)) * noise
a = lrn(500, 400, 60, 1e-9, 5)
kw = dict(epsilon=1e-7, b=16, seed=3)
f, t = E.iterative_cur(a, **kw)
o = O.iterative_cur(a, **kw)
print(compare_runs(o, f, t))
print('ranks', f.rank, o.rank, 'iters', len(t.rhos), len(o.rhos))
print('rhos eng', t.rhos); print('rhos orc', o.rhos)
print('err eng(LRt)', E.true_relative_error(a, f))
print('err orc(own idx)', O.true_relative_error(a, o.row_indices, o.col_indices))
print('err orc(eng idx)', O.true_relative_error(a, f.row_indices, f.col_indices))
C = a[:, f.col_indices]; R = a[f.row_indices, :]; X = a[np.ix_(f.row_indices, f.col_indices)]
print('cond X', np.linalg.cond(X))
print('err numpy lstsq', np.linalg.norm(a - C @ np.linalg.lstsq(X, R, rcond=None)[0]) / np.linalg.norm(a))
core = f.core_matrix()
print('err core', np.linalg.norm(a - C @ core @ R) / np.linalg.norm(a), 'core*X-I', np.linalg.norm(core @ X - np.eye(f.rank)))

"""Debug: engine vs oracle for wide blocks (b > 180) — first index difference and where it sits."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2509_21963_b200 as E  # noqa: E402
from oracle import oracle as O  # noqa: E402


def lrn(m, n, r, rel, seed):
    a = O.random_gaussian(m, r, seed) @ O.random_gaussian(n, r, seed + 1).T
    g = O.random_gaussian(m, n, seed + 2)
    return a + (rel * np.linalg.norm(a) / np.linalg.norm(g)) * g


a = lrn(1400, 1100, 420, 1e-12, 91)
for b in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "64,128,176,184,200,250").split(",")]:
    for sk in ("gaussian",):
        kw = dict(epsilon=1e-10, b=b, seed=4, sketch=sk)
        f, t = E.iterative_cur(a, **kw)
        o = O.iterative_cur(a, **kw)
        I, J = f.row_indices, f.col_indices
        d = next((q for q in range(min(len(J), o.rank)) if I[q] != o.row_indices[q] or J[q] != o.col_indices[q]), None)
        msg = f"b={b} {sk}: engine rank {f.rank} it {len(t.rhos)} {t.status}; oracle rank {o.rank} it {len(o.rhos)} {o.status}; first diff {d}"
        if d is not None:
            msg += f" (J {J[d]} vs {o.col_indices[d]}, I {I[d]} vs {o.row_indices[d]})"
            # engine steps vs oracle steps around the diff
            es = [(k, it, ix) for (k, it, ix, _, _) in t.steps]
            os_ = [(k, it, ix) for (k, it, ix, _, _) in o.steps]
            q = next((q for q in range(min(len(es), len(os_))) if es[q] != os_[q]), None)
            if q is not None:
                msg += f"; first step diff {q}: engine {es[q]} oracle {os_[q]} margin {o.steps[q][3]} {o.steps[q][4]}"
        print(msg, "rhos", [f"{x:.3e}" for x in t.rhos], [f"{x:.3e}" for x in o.rhos], flush=True)

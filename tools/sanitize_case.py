"""Small-shape workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every kernel family of the engine once — Gaussian DMMA sketch, sparse-sign mma.sync s8 and tcgen05
i8 sketches, the cluster / shared-memory / panel / global LUPP kernels, the lean and fused U-block
GEMMs, the wide-block solves, QRCP, the true error and the core export.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_21963_b200 as E  # noqa: E402
from paper_2509_21963_b200 import stages as S  # noqa: E402


def lrn(m, n, r, rel, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    g = rng.standard_normal((m, n))
    return a + (rel * np.linalg.norm(a) / np.linalg.norm(g)) * g


def run(a, **kw):
    f, t = E.iterative_cur(a, **kw)
    err = E.true_relative_error(a, f)
    core = f.core_matrix()
    print(f"{kw}: rank {f.rank} it {len(t.rhos)} {t.status} err {err:.2e} core {core.shape}", flush=True)


which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "engine"):
    run(lrn(600, 500, 40, 1e-9, 1), epsilon=1e-7, b=10, seed=0)                             # cluster LUPP, fused U block
    run(lrn(800, 400, 60, 1e-9, 2), epsilon=1e-6, b=20, seed=1, sketch="sparse_sign")       # mma.sync s8 sketch
    run(lrn(900, 700, 80, 1e-9, 3), epsilon=1e-7, b=40, seed=2, sketch="sparse_sign")       # tcgen05 i8 sketch
    run(lrn(700, 520, 100, 1e-10, 4), epsilon=1e-8, b=64, seed=3)                            # unfused GEMM + solves
    run(lrn(300, 260, 30, 1e-10, 5), epsilon=1e-8, b=8, seed=4, row_method="qrcp")          # QRCP rows, pivoted LU
    run(lrn(500, 450, 200, 1e-10, 6), epsilon=1e-6, b=200, seed=5)                          # wide block (global LU)
if which in ("all", "lupp"):
    for path in (1, 2, 3):  # cluster, grid shared-memory, panel/global
        r = S.time_lupp(3000, 20, reps=1, force_path=path)
        print("lupp path", path, r, flush=True)
if which in ("all", "gemm"):
    print("gemm", S.time_gemm(5000, 20, 300, reps=1), flush=True)
print("sanitize case done")

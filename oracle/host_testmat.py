"""BASELINE.json configs formed on the HOST (test infrastructure, like the rest of oracle/).

The CPU reference arm of bench.py (`--impl reference`) times the oracle on these matrices; it must
not load the engine (`paper_2509_21963_b200`, libitercur_b200.so) even to form its input, so the
recipes of paper_2509_21963_b200/testmat.py are restated here with the oracle's
Philox stream (bit-exact integer part, glibc log/cos — the reference's own rng.cpp arithmetic) and
numpy / torch-CPU BLAS for the products and QRs:

    cfg 1  2000 x 2000    U diag(10^(-(i-1)/20)) V^T
    cfg 2  20000 x 10000  U diag(i^-2) V^T
    cfg 3  50000 x 50000  RBF exp(-|x_i - y_j|^2 / (2 * 0.5^2)), x, y uniform on [0,1]^3
    cfg 4  100000^2       X diag(0.97^k) Y^T + 1e-10 G,  X, Y 100000 x 400, N(0, 1/400)
    cfg 5  200000 x 50000 X diag(k^-1.5) Y^T + 1e-6 G,   X 200000 x 1000, Y 50000 x 1000, N(0, 1/1000)

Streams: matrix seed 1, GenLeft = 4, GenRight = 5, GenNoise = 6 (proj/include/itercur/rng.hpp:16-18).
The device generator uses the same streams with correctly rounded log/cos and cuBLAS/cuSOLVER
products, so the two arms' matrices agree to rounding (same spectrum, same run shape), not bitwise;
parity tests copy the device matrix's bits instead (tools/parity_configs.py).
"""
from __future__ import annotations

import math

import numpy as np

from . import oracle as O

GEN_LEFT, GEN_RIGHT, GEN_NOISE = 4, 5, 6
MATRIX_SEED = 1

# == paper_2509_21963_b200/testmat.py CONFIGS (asserted equal by tests/test_host_testmat.py)
CONFIGS = {
    1: dict(m=2000, n=2000, sketch="gaussian", b=10, epsilon=1e-6, max_rank=0),
    2: dict(m=20000, n=10000, sketch="sparse_sign", b=20, epsilon=1e-4, max_rank=0),
    3: dict(m=50000, n=50000, sketch="gaussian", b=32, epsilon=1e-8, max_rank=0),
    4: dict(m=100000, n=100000, sketch="sparse_sign", b=50, epsilon=1e-6, max_rank=0),
    5: dict(m=200000, n=50000, sketch="gaussian", b=64, epsilon=1e-5, max_rank=1024),
}


def _gauss(rows, cols, stream, scale=1.0):
    out = np.empty((rows, cols), dtype=np.float64, order="F")
    O.gaussian_fill(out, MATRIX_SEED, stream, scale)
    return out


def generate(cfg: int, m: int | None = None, n: int | None = None) -> np.ndarray:
    """A for BASELINE config `cfg` as an (m, n) Fortran-ordered float64 host array. `m`, `n` shrink
    the shape for tests (same recipe)."""
    import torch

    c = CONFIGS[cfg]
    m = c["m"] if m is None else m
    n = c["n"] if n is None else n
    if cfg in (1, 2):
        u, _ = np.linalg.qr(_gauss(m, n, GEN_LEFT))
        v, _ = np.linalg.qr(_gauss(n, n, GEN_RIGHT))
        i = np.arange(1, n + 1, dtype=np.float64)
        sigma = 10.0 ** (-(i - 1) / 20.0) if cfg == 1 else i ** -2.0
        return np.asfortranarray((u * sigma) @ v.T)
    a = np.empty((m, n), dtype=np.float64, order="F")
    at = torch.from_numpy(a.T)  # (n, m) row-major view of the column-major A
    if cfg == 3:
        x = torch.tensor([[O.uniform_at(MATRIX_SEED, GEN_LEFT, i, d) for d in range(3)] for i in range(m)],
                         dtype=torch.float64)
        y = torch.tensor([[O.uniform_at(MATRIX_SEED, GEN_RIGHT, j, d) for d in range(3)] for j in range(n)],
                         dtype=torch.float64)
        chunk = max(1, (1 << 26) // m)
        for j0 in range(0, n, chunk):
            d2 = (y[j0:j0 + chunk, None, :] - x[None, :, :]).pow(2).sum(-1)
            at[j0:j0 + chunk] = torch.exp(-d2 / (2 * 0.5 ** 2))
        return a
    if cfg in (4, 5):
        k = 400 if cfg == 4 else 1000
        sd = math.sqrt(1.0 / k)
        xs = torch.from_numpy(_gauss(m, k, GEN_LEFT, sd))
        ys = torch.from_numpy(_gauss(n, k, GEN_RIGHT, sd))
        idx = torch.arange(1, k + 1, dtype=torch.float64)
        sigma = 0.97 ** idx if cfg == 4 else idx ** -1.5
        O.gaussian_fill(a, MATRIX_SEED, GEN_NOISE, 1e-10 if cfg == 4 else 1e-6)
        xsig = xs * sigma
        chunk = max(1, (1 << 30) // (8 * m))
        for j0 in range(0, n, chunk):
            at[j0:j0 + chunk] += ys[j0:j0 + chunk] @ xsig.t()
        return a
    raise ValueError(f"unknown config {cfg}")

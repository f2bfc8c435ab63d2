"""Test-only CPU backend for paper_2509_21963_b200.sharded (the product has no CPU path).

Implements the per-rank stage semantics of sharded.DeviceBackend in torch (CPU, float64)
and the oracle, so the multi-rank orchestration (exchanges, ownership, deterministic
reductions) can run under gloo with world_size > 1 on a machine without GPUs. The element
operations of the distributed LUPP step are the reference's (select.cpp:34-74: factor =
W(i,s)/pivot, W(i,t) -= factor*W(p,t), separately rounded), so the pivots are exact.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402  (test infrastructure)
from paper_2509_21963_b200.sharded import colmajor_empty, sketch_rows  # noqa: E402


class CpuBackend:
    device = torch.device("cpu")

    def sketch(self, a, b, seed, kind, nnz):
        y, ga, an = oracle.sketch(np.asfortranarray(a.numpy()), b, seed, kind, nnz)
        c = sketch_rows(b)
        cp = ((c + 7) // 8) * 8
        out = colmajor_empty(cp, a.shape[1], "cpu", fill=0.0)
        out[:c, :] = torch.from_numpy(np.ascontiguousarray(y))
        return out, ga * ga, an * an

    def lupp_step(self, W, live, steps, s, P, piv_local, row_offset, cand):
        rows = W.shape[0]
        if P is not None and 0 <= piv_local < rows:
            live[piv_local] = 0
        lv = live.bool()
        if P is not None:
            idx = lv.nonzero().squeeze(1)
            f = W[idx, s - 1] / P[s - 1]
            W[idx, s:steps] = W[idx, s:steps] - f[:, None] * P[None, s:steps]
        mags = W[:, s].abs().clone()
        mags[~lv] = -1.0
        cand.zero_()
        if rows == 0 or float(mags.max()) < 0.0:
            cand[0] = -1.0
            cand[1] = -1.0
            cand[2] = -1.0
            return
        i = int(torch.argmax(mags))  # first maximum: lowest index on ties
        others = torch.cat([mags[:i], mags[i + 1:]])
        cand[0] = mags[i]
        cand[1] = float(others.max()) if others.numel() else -1.0
        cand[2] = float(row_offset + i)
        cand[4 + s:4 + steps] = W[i, s:steps]

    def gemm(self, A, B, base, alpha, out):
        prod = A @ B if A.shape[1] else torch.zeros(out.shape, dtype=torch.float64)
        out.copy_((base if base is not None else 0.0) + alpha * prod)
        return out

    def select_columns(self, Y, b, pivot_floor, exclude):
        return oracle.select_columns(np.asfortranarray(Y.numpy()), b, pivot_floor=pivot_floor,
                                     exclude=exclude).indices

    def select_rows(self, S, b, pivot_floor, exclude):
        return oracle.select_rows(np.asfortranarray(S.numpy()), b, pivot_floor=pivot_floor, exclude=exclude).indices

    def block_lu(self, D):
        w = D.shape[0]
        for s in range(w):
            piv = D[s, s].clone()
            if s + 1 < w:
                f = D[s + 1:, s] / piv
                D[s + 1:, s + 1:] = D[s + 1:, s + 1:] - f[:, None] * D[s, s + 1:][None, :]
                D[s + 1:, s] = f
        return D

    def rows_solve(self, X, LU, out):
        w = LU.shape[0]
        x = X.clone()
        for q in range(1, w):
            for p in range(q):
                x[:, q] = x[:, q] - LU[q, p] * x[:, p]
        for q in range(w - 1, -1, -1):
            for p in range(q + 1, w):
                x[:, q] = x[:, q] - LU[q, p] * x[:, p]
            x[:, q] = x[:, q] / LU[q, q]
        out.copy_(x)
        return out

"""Column-sharded IterativeCUR across ranks, one process per GPU.

Each rank owns a contiguous column range A(:, off:off+n_r) of A (column-major, so the shard
is contiguous memory). The algorithm is the single-device one (csrc/engine.cu; the
reference's proj/src/driver.cpp:48-167 in incremental block-LU form) with the exchanges the
sharding needs:

  step                                   data on each rank            exchange per call
  sketch Y_r = S·A_r, ||A_r||², ||Y_r||²   S from (seed, i, j)          all_reduce of 2 doubles
  column LUPP on Y^T (b pivot steps)      rows of Y^T = own columns     per step: all_gather of the
                                                                       candidates (|v|, 2nd, index,
                                                                       row tail), reduced in rank
                                                                       order = lowest index on ties
  A(:,J_k), R~(:,J_k), Y(:,J_k)           owners contribute            all_reduce (sum of disjoint
                                                                       contributions: exact)
  S_row = A(:,J_k) − L·R~(:,J_k), row     replicated (identical bits    none
  LUPP, D_k = LU(S_row(I_k,:))            on every rank)
  U_k, R~_k rows, Y_r −= Y(:,J_k)·R~_k     local to the shard            all_reduce of ||Y_r||²

I and J are identical to the single-device run unless a ρ or floor comparison sits within
rounding of its threshold (the norms are sums over shards in a different order).

Two executions of this protocol:

* the product path (`iterative_cur_sharded` on CUDA tensors, no `backend`): the whole loop runs in
  the C++ engine (csrc/engine.cu, itercur_iterative_cur_sharded_device) over an NCCL communicator
  built for the torch.distributed group, every collective enqueued on the run's stream and
  captured in its iteration graphs — no host round trip per iteration. The column selection
  replicates Y^T(:, 0:b) (one in-place allgather per iteration) instead of exchanging candidates
  per pivot step, and the engine requires the standard block partition (`shard_range`);
* the protocol model (a `backend` is passed): this module's Python loop over per-rank stages with
  torch.distributed collectives — both column exchanges ("sketch", "candidates") — run on CPU with
  gloo and a test-only backend (tests/sharded_cpu_backend.py) and on the B200 stage kernels
  (`DeviceBackend`). It is the executable specification the native path is checked against.

`iterative_cur_emulated_shards` runs the native sharded pipeline with all shards in one process on
one GPU (per-shard kernels, collectives as device writes): the multi-rank data path on one device.
The product has no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from . import _capi
from ._capi import check as _check

_SKETCHES = {"gaussian": 0, "sparse_sign": 1}
_STATUS = {0: "Converged", 1: "MaxRank", 2: "ResidualExhausted"}
_EPS = 2.220446049250313e-16


def sketch_rows(b: int) -> int:
    return (11 * int(b)) // 10  # proj/include/itercur/sketch.hpp:10


def _even(x: int) -> int:
    return x + (x & 1)


def colmajor_empty(rows: int, cols: int, device, dtype=torch.float64, fill=None) -> torch.Tensor:
    """(rows, cols) view with column-major strides (1, ld), ld even (16-byte aligned columns)."""
    ld = max(_even(rows), 2)
    base = torch.empty(max(cols, 1), ld, dtype=dtype, device=device) if fill is None else \
        torch.full((max(cols, 1), ld), fill, dtype=dtype, device=device)
    return base.t()[:rows, :cols]


def to_colmajor(t: torch.Tensor) -> torch.Tensor:
    out = colmajor_empty(t.shape[0], t.shape[1], t.device, t.dtype)
    out.copy_(t)
    return out


def _ld(t: torch.Tensor) -> int:
    if t.dim() != 2 or (t.shape[0] > 1 and t.stride(0) != 1):
        raise ValueError("expected a column-major 2-D tensor")
    return int(t.stride(1)) if t.shape[1] > 1 else max(_even(t.shape[0]), 2)


class DeviceBackend:
    """Per-rank stages on this rank's GPU (libitercur_b200.so kernels)."""

    def __init__(self, device):
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise RuntimeError("DeviceBackend needs a CUDA device: the B200 engine has no CPU path")
        self.lib = _capi.lib()

    def _st(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def sketch(self, a, b, seed, kind, nnz):
        m, n = a.shape
        c = sketch_rows(b)
        cp = ((c + 7) // 8) * 8
        yc = torch.empty(n, max(c, 1), dtype=torch.float64, device=self.device)  # c x n, ld = c (the C-ABI layout)
        ga, an = C.c_double(), C.c_double()
        _check(self.lib.itercur_sketch_device(C.c_void_p(a.data_ptr()), m, n, _ld(a), int(b), int(seed),
                                              _SKETCHES[kind], int(nnz), C.c_void_p(yc.data_ptr()), C.byref(ga),
                                              C.byref(an), self._st()))
        y = colmajor_empty(cp, n, self.device, fill=0.0)
        y[:c, :].copy_(yc.t()[:c, :])
        return y, ga.value ** 2, an.value ** 2

    def lupp_step(self, W, live, steps, s, P, piv_local, row_offset, cand):
        _check(self.lib.itercur_lupp_dist_step(C.c_void_p(W.data_ptr()), W.shape[0], _ld(W), int(steps), int(s),
                                               C.c_void_p(P.data_ptr() if P is not None else 0), int(piv_local),
                                               C.c_void_p(live.data_ptr()), int(row_offset),
                                               C.c_void_p(cand.data_ptr()), self._st()))

    def gemm(self, A, B, base, alpha, out):
        """out = base + alpha * A @ B (all column-major)."""
        M, K = A.shape
        N = B.shape[1]
        if K == 0:
            out.copy_(base if base is not None else torch.zeros_like(out))
            return out
        _check(self.lib.itercur_gemm_device(M, N, K, C.c_void_p(A.data_ptr()), _ld(A), C.c_void_p(B.data_ptr()),
                                            _ld(B), C.c_void_p(base.data_ptr() if base is not None else 0),
                                            _ld(base) if base is not None else 0, float(alpha),
                                            C.c_void_p(out.data_ptr()), _ld(out), self._st()))
        return out

    def select_columns(self, Y, b, pivot_floor, exclude):
        from .stages import select_columns
        return select_columns(Y, b, pivot_floor=pivot_floor, exclude=exclude).indices

    def select_rows(self, S, b, pivot_floor, exclude):
        from .stages import select_rows
        sel = select_rows(S, b, pivot_floor=pivot_floor, exclude=exclude)
        return sel.indices

    def block_lu(self, D):
        _check(self.lib.itercur_block_lu_device(C.c_void_p(D.data_ptr()), D.shape[0], _ld(D), self._st()))
        return D

    def rows_solve(self, X, LU, out):
        _check(self.lib.itercur_rows_lu_solve_device(C.c_void_p(X.data_ptr()), _ld(X), X.shape[0],
                                                     C.c_void_p(LU.data_ptr()), _ld(LU), LU.shape[0],
                                                     C.c_void_p(out.data_ptr()), _ld(out), self._st()))
        return out


@dataclass
class ShardedResult:
    row_indices: list
    col_indices: list
    status: str
    final_rho: float
    threshold: float
    rhos: list = field(default_factory=list)
    note: str = ""
    col_steps: list = field(default_factory=list)  # (index, |best|, runner-up) per column pivot step
    exchanges: int = 0                              # collectives issued by this rank
    native: object = None                           # the C++ run (product path)
    kernel_launches: int = 0

    @property
    def rank(self) -> int:
        return len(self.row_indices)


class _Comm:
    def __init__(self, group):
        self.group = group
        self.on = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.on else 1
        self.rank = dist.get_rank(group) if self.on else 0
        self.count = 0

    def all_reduce(self, t):
        if self.world > 1:
            if t.is_contiguous():
                dist.all_reduce(t, group=self.group)
            else:  # column-major views: reduce a dense copy
                buf = t.contiguous()
                dist.all_reduce(buf, group=self.group)
                t.copy_(buf)
            self.count += 1
        return t

    def all_gather(self, t):
        if self.world == 1:
            return t.unsqueeze(0)
        flat = torch.empty(self.world * t.numel(), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(flat, t.contiguous().view(-1), group=self.group)
        self.count += 1
        return flat.view((self.world,) + tuple(t.shape))

    def all_gather_obj(self, v):
        if self.world == 1:
            return [v]
        out = [None] * self.world
        dist.all_gather_object(out, v, group=self.group)
        self.count += 1
        return out


def _gather_columns(comm, y, widths):
    """Y_full = [Y_0 | Y_1 | ...] (c_pad x n, column-major) from every rank's c_pad x n_r block:
    one all_gather of equal-size (padded) flat buffers."""
    cp = y.shape[0]
    if comm.world == 1:
        return y
    maxn = max(widths)
    buf = torch.zeros(maxn * cp, dtype=y.dtype, device=y.device)
    n_r = y.shape[1]
    if n_r:
        buf[:n_r * cp].view(n_r, cp).copy_(y.t())
    g = comm.all_gather(buf)                                  # world x (maxn * cp)
    parts = [g[q, :widths[q] * cp] for q in range(comm.world)]
    return torch.cat(parts).view(sum(widths), cp).t()


def _dist_column_lupp(be, comm, y, col_live, steps, ynorm, pivot_floor, col_offset, n_r, col_steps):
    """Distributed LUPP on W = Y^T (select.cpp:34-74, 121-139): every rank eliminates its own rows;
    one all_gather of the per-rank pivot candidates per step, reduced in rank order (lowest global
    index on ties)."""
    dev = y.device
    W = to_colmajor(y[:steps, :].t())                # n_r x steps
    live = col_live.clone()
    cand = torch.zeros(4 + steps, dtype=torch.float64, device=dev)
    abs_floor = 1e2 * _EPS * ynorm
    cols, P, piv_local, first = [], None, -1, 0.0
    for s in range(steps):
        if n_r:
            be.lupp_step(W, live, steps, s, P, piv_local, col_offset, cand)
        else:
            cand.zero_()
            cand[0] = -1.0
        g = comm.all_gather(cand)                     # world x (4 + steps)
        mags = g[:, 0]
        wr = int(torch.argmax(mags).item())           # first maximum in rank order
        best = float(mags[wr])
        if best < 0.0 or best <= abs_floor:
            break
        if s == 0:
            first = best
        elif best < pivot_floor * first:
            break
        others = torch.cat([mags[:wr], mags[wr + 1:]])
        second = max(float(g[wr, 1]), float(others.max()) if others.numel() else -1.0)
        idx = int(g[wr, 2])
        cols.append(idx)
        col_steps.append((idx, best, second))
        P = g[wr, 4:].contiguous()
        piv_local = idx - col_offset if wr == comm.rank else -1
    return cols


# ------------------------------------------------------------------ native (C++ / NCCL) path
def shard_range(n_total: int, world: int, rank: int):
    """(offset, count) of rank's column block in the engine's partition (blocks of even width)."""
    off, cnt = C.c_int64(), C.c_int64()
    _check(_capi.lib().itercur_shard_range(int(n_total), int(world), int(rank), C.byref(off), C.byref(cnt)))
    return off.value, cnt.value


_COMMS = {}


def native_comm(group=None):
    """The engine's NCCL communicator over the ranks of a torch.distributed group (created once per
    group on this rank's current device; the unique id travels through torch.distributed)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    key = (id(group), world, torch.cuda.current_device())
    if key in _COMMS:
        return _COMMS[key], world, rank
    L = _capi.lib()
    uid = (C.c_char * 128)()
    if rank == 0:
        _check(L.itercur_nccl_unique_id(uid))
    if world > 1:
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        C.memmove(uid, box[0], 128)
    comm = C.c_void_p()
    # NCCL prints its version banner on stdout at init: keep stdout clean for callers that emit
    # machine-read lines there (bench.py), routing the banner to stderr
    import os
    import sys

    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        rc = L.itercur_nccl_comm_init(world, uid, rank, C.byref(comm))
    finally:
        os.dup2(saved, 1)
        os.close(saved)
    _check(rc)
    _COMMS[key] = comm
    return comm, world, rank


def _native_config(b, epsilon, delta, alpha, risk_adjust, max_rank, max_iters, pivot_floor, seed, sketch,
                   sparse_nnz):
    from . import _config

    return _config(epsilon, b, delta, alpha, risk_adjust, max_rank, max_iters, "lupp", "lupp", pivot_floor, seed,
                   sketch, sparse_nnz, False)


def _native_result(run_ptr, keep):
    from . import _collect

    f, t = _collect(run_ptr, keep)
    return ShardedResult(f.row_indices, f.col_indices, t.status, t.final_rho, t.threshold, t.rhos, t.note,
                         [(ix, b, s) for (k, _, ix, b, s) in t.steps if k == 0], 0, f, t.kernel_launches)


def _native_sharded(a, col_offset, n_total, cfg, group):
    m, n_r = a.shape
    comm, world, rank = native_comm(group)
    off, cnt = shard_range(n_total, world, rank)
    if off != col_offset or cnt != n_r:
        raise ValueError(f"rank {rank} of {world} must hold columns [{off}, {off + cnt}) of the {n_total} "
                         f"(shard_range); got [{col_offset}, {col_offset + n_r})")
    out = C.c_void_p()
    with torch.cuda.device(a.device):
        stream = torch.cuda.current_stream(a.device).cuda_stream
        _check(_capi.lib().itercur_iterative_cur_sharded_device(C.c_void_p(a.data_ptr()), m, n_r, _ld(a), int(n_total),
                                                                C.byref(cfg), comm, C.c_void_p(stream),
                                                                C.byref(out)))
    return _native_result(out.value, a)


def iterative_cur_emulated_shards(a: torch.Tensor, shards: int, *, epsilon=1e-6, b=50, delta=0.0, alpha=0.05,
                                  risk_adjust=False, max_rank=0, max_iters=0, pivot_floor=1e-13, seed=0,
                                  sketch="gaussian", sparse_nnz=8):
    """The native column-sharded pipeline with `shards` shards computed on this one device (the
    collectives become the equivalent device writes); returns (CurFactors, RunTrace) like
    `iterative_cur` — exports work, every shard being local."""
    from . import _collect

    cfg = _native_config(b, epsilon, delta, alpha, risk_adjust, max_rank, max_iters, pivot_floor, seed, sketch,
                         sparse_nnz)
    m, n = a.shape
    out = C.c_void_p()
    with torch.cuda.device(a.device):
        stream = torch.cuda.current_stream(a.device).cuda_stream
        _check(_capi.lib().itercur_iterative_cur_sharded_emulated(C.c_void_p(a.data_ptr()), m, n, _ld(a), int(shards),
                                                                  C.byref(cfg), C.c_void_p(stream), C.byref(out)))
    return _collect(out.value, a)


def iterative_cur_sharded(a_shard: torch.Tensor, col_offset: int, n_total: int, *, epsilon=1e-6, b=50, delta=0.0,
                          alpha=0.05, risk_adjust=False, max_rank=0, max_iters=0, pivot_floor=1e-13, seed=0,
                          sketch="gaussian", sparse_nnz=8, group=None, backend=None,
                          column_exchange="sketch") -> ShardedResult:
    """IterativeCUR of A = [A_0 | A_1 | ...] with this rank's block `a_shard` = A(:, col_offset :
    col_offset + n_r) (column-major, on this rank's device). Collective: every rank of `group`
    calls it with its own shard; all ranks return the same indices and trace.

    Without a `backend` (CUDA shards) this is the native C++ engine over NCCL (the block must be
    `shard_range(n_total, world, rank)`). With a `backend`, the Python protocol model runs:
    column_exchange "sketch" (default) replicates the c_pad x n sketch once per iteration and runs
    the column LUPP whole on every rank (2 collectives per iteration); "candidates" runs the
    distributed LUPP (one all_gather of pivot candidates per pivot step)."""
    if backend is None and a_shard.is_cuda and column_exchange == "sketch":
        if sketch not in _SKETCHES:
            raise ValueError(f"unknown sketch kind '{sketch}'")
        a = a_shard if (a_shard.shape[0] <= 1 or a_shard.stride(0) == 1) and _ld(a_shard) % 2 == 0 \
            else to_colmajor(a_shard)
        cfg = _native_config(b, epsilon, delta, alpha, risk_adjust, max_rank, max_iters, pivot_floor, seed, sketch,
                             sparse_nnz)
        return _native_sharded(a, int(col_offset), int(n_total), cfg, group)
    if column_exchange not in ("sketch", "candidates"):
        raise ValueError(f"unknown column_exchange '{column_exchange}'")
    comm = _Comm(group)
    dev = a_shard.device
    be = backend if backend is not None else DeviceBackend(dev)
    a = a_shard if (a_shard.shape[0] <= 1 or a_shard.stride(0) == 1) and _ld(a_shard) % 2 == 0 \
        else to_colmajor(a_shard)
    m, n_r = a.shape
    # every shard must describe the same problem (contiguous column ranges in rank order)
    shapes = comm.all_gather_obj((int(m), int(col_offset), int(n_r)))
    if any(sh[0] != m for sh in shapes) or sum(sh[2] for sh in shapes) != n_total or \
            any(shapes[q][1] != sum(sh[2] for sh in shapes[:q]) for q in range(len(shapes))):
        raise ValueError("shards must be contiguous column ranges of one m x n matrix, in rank order")
    n = int(n_total)
    if m == 0 or n == 0:
        raise ValueError("matrix must be nonempty")
    if sketch not in _SKETCHES:
        raise ValueError(f"unknown sketch kind '{sketch}'")

    c = sketch_rows(b)
    # ---- sketch + norms (make_sketch, sketch.cpp:10-24; driver.cpp:51-54) ----
    if epsilon < 0.0 or b < 1 or b > m:
        y, ysq_r, asq_r = None, 0.0, float((a.double() ** 2).sum().item()) if n_r else 0.0
    else:
        y, ysq_r, asq_r = be.sketch(a, b, seed, sketch, sparse_nnz) if n_r else \
            (colmajor_empty(((c + 7) // 8) * 8, 0, dev), 0.0, 0.0)
    sums = comm.all_reduce(torch.tensor([ysq_r, asq_r], dtype=torch.float64, device=dev))
    ysq, asq = float(sums[0]), float(sums[1])
    if not math.isfinite(asq):
        raise ValueError("matrix contains non-finite entries")
    if asq == 0.0:
        raise ValueError("matrix must be nonzero")
    if epsilon < 0.0:
        raise ValueError("epsilon must be nonnegative")
    if b < 1:
        raise ValueError("block size must be at least 1")
    if b > m:
        raise ValueError("block exceeds row count")
    if not (0.0 < pivot_floor < 1.0):
        raise ValueError("pivot_floor must lie in (0, 1)")
    ga_norm = math.sqrt(ysq)
    min_dim = min(m, n)
    max_rank_eff = min(max_rank, min_dim) if max_rank > 0 else min_dim
    max_iters_eff = max_iters if max_iters > 0 else (min_dim + b - 1) // b + 1
    if risk_adjust:
        from . import adjusted_threshold
        threshold = adjusted_threshold(epsilon, delta, alpha, c)
    else:
        threshold = epsilon
    ynorm = ga_norm  # ||Y||_F of the current column residual (the column LUPP's floor, select.cpp:127)
    rho = 1.0 if ga_norm > 0.0 else 0.0
    if rho <= threshold:
        return ShardedResult([], [], "Converged", rho, threshold, [],
                             "threshold at or above the initial estimate; empty factorization", [], comm.count)

    widths = [sh[2] for sh in shapes]
    yfull = _gather_columns(comm, y, widths) if column_exchange == "sketch" else None
    cap = max_rank_eff + b
    L = colmajor_empty(m, cap, dev, fill=0.0)             # residual columns, replicated
    RtT = colmajor_empty(n_r, cap, dev, fill=0.0)         # R~^T for this shard (n_r x cap, column-major)
    col_live = torch.ones(n_r, dtype=torch.uint8, device=dev)
    I, J, rhos, col_steps = [], [], [], []
    r, k = 0, 0
    status = "MaxRank"
    while True:
        if r >= max_rank_eff or k >= max_iters_eff:
            status = "MaxRank"
            break
        block = min(b, max_rank_eff - r)
        # ---- column selection (select.cpp:121-139) ----
        steps = min(block, c)
        if column_exchange == "sketch":
            # Y is replicated once per iteration (one all_gather of c_pad x n_r per rank); every
            # rank then runs the single-device LUPP on the whole Y^T: same pivots on every rank,
            # no per-step exchange.
            sel = be.select_columns(yfull[:c, :], steps, pivot_floor, J)
            cols = list(sel)[:steps]
        else:
            cols = _dist_column_lupp(be, comm, y, col_live, steps, ynorm, pivot_floor, col_offset, n_r, col_steps)
        if not cols:
            status = "ResidualExhausted"
            break
        w_cols = len(cols)
        own = [(q, j - col_offset) for q, j in enumerate(cols) if col_offset <= j < col_offset + n_r]
        # ---- A(:,J_k), R~(:,J_k) (and Y(:,J_k) unless Y is replicated) from their owners: one all_reduce
        # of disjoint contributions (exact) ----
        yrows = y.shape[0] if column_exchange != "sketch" else 0
        pack = torch.zeros(w_cols, _even(m + r + yrows), dtype=torch.float64, device=dev)  # column q = [A; R~; Y](:, J_q)
        if own:
            qs = torch.tensor([q for q, _ in own], dtype=torch.int64, device=dev)
            js = torch.tensor([jl for _, jl in own], dtype=torch.int64, device=dev)
            pack[qs, :m] = a.index_select(1, js).t()
            if r:
                pack[qs, m:m + r] = RtT[:, :r].index_select(0, js)
            if yrows:
                pack[qs, m + r:m + r + yrows] = y.index_select(1, js).t()
        comm.all_reduce(pack)
        packT = pack.t()                                  # (m + r + yrows) x w, column-major view
        Acols = packT[:m, :]
        Rcols = to_colmajor(packT[m:m + r, :]) if r else colmajor_empty(1, w_cols, dev, fill=0.0)
        if yrows:
            Ycols = to_colmajor(packT[m + r:m + r + yrows, :])
        else:
            Jk_t = torch.tensor(cols, dtype=torch.int64, device=dev)
            Ycols = yfull[:, Jk_t]
        # ---- row residual S_row = A(:,J_k) - L R~(:,J_k) (replicated; sketch.cpp:43-60) ----
        S = colmajor_empty(m, w_cols, dev)
        be.gemm(L[:, :r], Rcols[:r, :], Acols, -1.0, S)
        rows = be.select_rows(S, w_cols, pivot_floor, I)  # select.cpp:141-165, replicated
        if not rows:
            status = "ResidualExhausted"
            break
        width = min(w_cols, len(rows))
        Ik, Jk = rows[:width], cols[:width]
        L[:, r:r + width].copy_(S[:, :width])
        Ik_t = torch.tensor(Ik, dtype=torch.int64, device=dev)
        D = to_colmajor(S[Ik_t, :width])
        be.block_lu(D)
        if bool(torch.any(torch.diagonal(D) == 0.0).item()):
            status = "ResidualExhausted"  # singular cross block (pinv.cpp:50-52 -> driver.cpp:135-139)
            break
        # ---- U block and R~ rows of this shard: U_k^T = A(I_k,:)^T - R~^T L(I_k,:)^T ----
        if n_r:
            At = to_colmajor(a[Ik_t, :].t())            # n_r x width
            Ut = colmajor_empty(n_r, width, dev)
            be.gemm(RtT[:, :r], to_colmajor(L[Ik_t, :r].t()), At, -1.0, Ut)
            Rk = RtT[:, r:r + width]                     # R~_k^T solved in place of its columns
            be.rows_solve(Ut, D, Rk)
            # ---- downdate Y^T -= R~_k^T Y(:,J_k)^T (sketch.cpp:26-41) ----
            Yt = to_colmajor(y.t())                      # n_r x cp
            Ynew = colmajor_empty(n_r, y.shape[0], dev)
            be.gemm(Rk, to_colmajor(Ycols[:, :width].t()), Yt, -1.0, Ynew)
            y = to_colmajor(Ynew.t())
        if column_exchange != "sketch":
            for q, jl in own:
                if q < width:
                    col_live[jl] = 0
        if column_exchange == "sketch":
            yfull = _gather_columns(comm, y, widths)
            ysq_all = float(torch.sum(yfull[:c, :] * yfull[:c, :]).item())
        else:
            ysq_r = float((y.double() ** 2).sum().item()) if n_r else 0.0
            ysq_all = float(comm.all_reduce(torch.tensor([ysq_r], dtype=torch.float64, device=dev))[0])
        ynorm = math.sqrt(ysq_all)
        rho = ynorm / ga_norm if ga_norm > 0 else 0.0
        I += Ik
        J += Jk
        r += width
        rhos.append(rho)
        k += 1
        if rho <= threshold:
            status = "Converged"
            break
    return ShardedResult(I, J, status, rho, threshold, rhos, "", col_steps, comm.count)


def true_relative_error_sharded(a_shard: torch.Tensor, col_offset: int, result: ShardedResult, group=None,
                                backend=None) -> float:
    """||A - C U R||_F / ||A||_F with the column sums of squares reduced over the shards
    (driver.cpp:169-190); C U R = C X^{-1} R with X = A(I, J). A native result evaluates on the
    engine (collective over its communicator: ||A_s - L R~_s||^2 per rank, summed)."""
    if result.native is not None and backend is None:
        out = C.c_double()
        _check(_capi.lib().itercur_true_relative_error_sharded(result.native._run.ptr, C.byref(out)))
        return out.value
    comm = _Comm(group)
    dev = a_shard.device
    a = a_shard
    m, n_r = a.shape
    asq = comm.all_reduce(torch.tensor([float((a.double() ** 2).sum().item())], dtype=torch.float64, device=dev))
    if float(asq[0]) == 0.0:
        return 0.0
    if not result.row_indices:
        return 1.0
    I = torch.tensor(result.row_indices, dtype=torch.int64, device=dev)
    own = [(q, j - col_offset) for q, j in enumerate(result.col_indices) if col_offset <= j < col_offset + n_r]
    Cm = torch.zeros(m, len(result.col_indices), dtype=torch.float64, device=dev)
    for q, jl in own:
        Cm[:, q] = a[:, jl]
    comm.all_reduce(Cm)
    X = Cm[I, :]
    Rm = a[I, :].double()
    diff = a.double() - Cm @ torch.linalg.solve(X, Rm)
    sq = comm.all_reduce(torch.tensor([float((diff ** 2).sum().item())], dtype=torch.float64, device=dev))
    return math.sqrt(float(sq[0])) / math.sqrt(float(asq[0]))

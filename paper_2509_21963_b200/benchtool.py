"""The reference's experiment harness on the B200 engine (proj/src/bench.cpp,
proj/include/itercur/bench.hpp, CLI proj/tools/benchcli_main.cpp):

    python -m paper_2509_21963_b200.benchtool threshold --matrix gen:lowrank:2000,1500,40 \
        --b 20 --eps 1e-6 --reps 3 --seed 0 --out threshold.csv

Sources (`load_matrix`, bench.cpp:90-135): gen:lowrank:M,N,R | gen:lowrankpd:M,N,R[,DECAY] |
gen:lehmer:N | gen:expdecay:N,RATIO (formed on the device, testmat.py) and mm:<path>
(MatrixMarket, mmio.py). Every experiment times only the algorithm call with a steady clock
(bench.cpp:18-22, 160-162) and writes the reference's CSV layout with %.17g values and %.6f
times (bench.cpp:24-34). The algorithm calls are the engine's (iterative_cur, slupp_cur,
true_relative_error, sketched_relative_error); only the TSVD reference rows of fixed-rank /
selection use a library SVD (Eigen BDCSVD in the reference, baselines.cpp:19-33).
"""
from __future__ import annotations

import argparse
import math
import re
import sys
import time
from dataclasses import dataclass, field

from . import MatrixHandle, iterative_cur, slupp_cur, sketched_relative_error, true_relative_error
from . import testmat

_INT = re.compile(r"^\s*[+-]?\d+$")
_FLOAT_PREFIX = re.compile(r"^\s*[+-]?(?:inf(?:inity)?|nan|(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?)", re.IGNORECASE)


@dataclass
class ExperimentConfig:
    """proj/include/itercur/bench.hpp:14-30."""
    kind: str = "threshold"
    matrix_source: str = ""
    b: int = 50
    epsilon: float = 1e-6
    delta: float = 0.0
    alpha: float = 0.05
    risk_adjust: bool = False
    ranks: list = field(default_factory=list)
    blocks: list = field(default_factory=list)
    reps: int = 1
    seed_base: int = 0
    out_path: str = ""
    deterministic: bool = False


def _tokens(args: str):
    """std::getline(ss, token, ',') splitting: no trailing empty token."""
    parts = args.split(",")
    if parts and parts[-1] == "":
        parts.pop()
    return parts


def _parse_index_args(args, lo, hi, source):
    """bench.cpp:43-60."""
    out = []
    for tok in _tokens(args):
        if not _INT.match(tok):
            raise ValueError(f"bad generator argument '{tok}' in '{source}'")
        out.append(int(tok))
    if len(out) < lo or len(out) > hi:
        raise ValueError(f"wrong number of generator arguments in '{source}'")
    return out


def _stod(tok: str) -> float:
    """std::stod: the longest numeric prefix (no full-consumption check)."""
    mt = _FLOAT_PREFIX.match(tok)
    if not mt:
        raise ValueError("stod")
    return float(mt.group(0))


def load_matrix(source: str, seed: int, device="cuda") -> MatrixHandle:
    """bench.cpp:90-135."""
    if source.startswith("mm:"):
        from .mmio import read_matrix_market

        return read_matrix_market(source[3:])
    if not source.startswith("gen:"):
        raise ValueError("matrix source must start with 'gen:' or 'mm:'")
    rest = source[4:]
    colon = rest.find(":")
    if colon < 0:
        raise ValueError(f"generator spec '{source}' needs arguments")
    kind, args = rest[:colon], rest[colon + 1:]
    if kind == "lowrank":
        m, n, r = _parse_index_args(args, 3, 3, source)
        return MatrixHandle.device(testmat.low_rank(m, n, r, seed, device=device))
    if kind == "lowrankpd":
        parts = _tokens(args)
        if len(parts) not in (3, 4):
            raise ValueError(f"wrong number of generator arguments in '{source}'")
        m, n, r = _parse_index_args(",".join(parts[:3]), 3, 3, source)
        decay = _stod(parts[3]) if len(parts) == 4 else 0.0
        return MatrixHandle.device(testmat.low_rank_pd(m, n, r, decay, seed, device=device))
    if kind == "lehmer":
        (n,) = _parse_index_args(args, 1, 1, source)
        return MatrixHandle.device(testmat.lehmer(n, device=device))
    if kind == "expdecay":
        parts = _tokens(args)
        if len(parts) != 2:
            raise ValueError(f"wrong number of generator arguments in '{source}'")
        (n,) = _parse_index_args(parts[0], 1, 1, source)
        return MatrixHandle.device(testmat.exp_decay(n, _stod(parts[1]), seed, device=device))
    raise ValueError(f"unknown generator kind '{kind}'")


def _fmt_value(v: float) -> str:
    return "%.17g" % v


def _fmt_time(v: float) -> str:
    return "%.6f" % v


def _emit(cfg: ExperimentConfig, csv: str) -> None:
    if not cfg.out_path:
        return
    try:
        with open(cfg.out_path, "w") as f:
            f.write(csv)
    except OSError as e:
        raise RuntimeError(f"cannot open '{cfg.out_path}' for writing") from e


def _validate_common(cfg):
    if cfg.reps < 1:
        raise ValueError("repetitions must be at least 1")


def _validate_ranks(cfg, a: MatrixHandle):
    if not cfg.ranks:
        raise ValueError("rank list must not be empty")
    if list(cfg.ranks) != sorted(cfg.ranks):
        raise ValueError("rank list must be sorted ascending")
    min_dim = min(a.rows, a.cols)
    for r in cfg.ranks:
        if r < 1:
            raise ValueError("ranks must be positive")
        if r > min_dim:
            raise ValueError(f"rank {r} exceeds min(m, n) = {min_dim}")


def _pure_rank(b, rank):
    """bench.cpp:80-86: epsilon 0, max_rank = rank."""
    return dict(epsilon=0.0, b=int(b), max_rank=int(rank))


def _tail_energies(a: MatrixHandle):
    """compute_spectrum (baselines.cpp:19-33): tail_energies[i] = ||sigma[i:]||."""
    import torch

    t = a._densified_on_device()._tensor if a.is_sparse else (a._tensor if a.is_device else
                                                             torch.from_numpy(a.to_numpy()).cuda())
    s = torch.linalg.svdvals(t).double().cpu().numpy()
    tails = [0.0] * (len(s) + 1)
    sq = 0.0
    for i in range(len(s) - 1, -1, -1):
        sq += s[i] * s[i]
        tails[i] = math.sqrt(sq)
    return tails


def run_threshold(cfg: ExperimentConfig) -> str:
    """bench.cpp:137-190: adaptive runs to the tolerance vs the s-LUPP baseline at the found rank."""
    _validate_common(cfg)
    a = load_matrix(cfg.matrix_source, cfg.seed_base)
    rows = []
    for rep in range(cfg.reps):
        seed = cfg.seed_base + rep
        t0 = time.perf_counter()
        f, t = iterative_cur(a, epsilon=cfg.epsilon, b=cfg.b, delta=cfg.delta, alpha=cfg.alpha,
                             risk_adjust=cfg.risk_adjust, seed=seed)
        wall = time.perf_counter() - t0
        rows.append(("IterativeCUR", rep, f.rank, true_relative_error(a, f), t.final_rho, wall))
        t0 = time.perf_counter()
        base = slupp_cur(a, f.rank, seed)
        wall = time.perf_counter() - t0
        # the adaptive run's estimator sketch scores the baseline (bench.cpp:171-174)
        sketched = sketched_relative_error(a, base, cfg.b, seed)
        rows.append(("s-LUPP", rep, base.rank, true_relative_error(a, base), sketched, wall))
    rows.sort(key=lambda r: (r[0], r[1]))
    csv = "method,rep,final_rank,rel_error_true,rel_error_sketched,wall_time_s\n" + "".join(
        f"{m},{rep},{rank},{_fmt_value(et)},{_fmt_value(es)},{_fmt_time(w)}\n" for m, rep, rank, et, es, w in rows)
    _emit(cfg, csv)
    return csv


def run_fixed_rank(cfg: ExperimentConfig) -> str:
    """bench.cpp:192-240."""
    _validate_common(cfg)
    a = load_matrix(cfg.matrix_source, cfg.seed_base)
    _validate_ranks(cfg, a)
    a_norm = a.fro_norm()
    t0 = time.perf_counter()
    tails = _tail_energies(a)
    svd_wall = time.perf_counter() - t0
    rows = []
    for rank in cfg.ranks:
        rows.append(("TSVD", rank, 0, (tails[rank] if rank < len(tails) else 0.0) / a_norm, svd_wall))
        for rep in range(cfg.reps):
            seed = cfg.seed_base + rep
            t0 = time.perf_counter()
            f, _ = iterative_cur(a, seed=seed, **_pure_rank(cfg.b, rank))
            wall = time.perf_counter() - t0
            rows.append(("IterativeCUR", rank, rep, true_relative_error(a, f), wall))
            t0 = time.perf_counter()
            base = slupp_cur(a, rank, seed)
            wall = time.perf_counter() - t0
            rows.append(("s-LUPP", rank, rep, true_relative_error(a, base), wall))
    rows.sort(key=lambda r: (r[0], r[1], r[2]))
    csv = "method,rank,rep,rel_error,wall_time_s\n" + "".join(
        f"{m},{rank},{rep},{_fmt_value(e)},{_fmt_time(w)}\n" for m, rank, rep, e, w in rows)
    _emit(cfg, csv)
    return csv


def run_selection_methods(cfg: ExperimentConfig) -> str:
    """bench.cpp:242-280: LUPP vs QRCP selection over the rank grid."""
    _validate_common(cfg)
    a = load_matrix(cfg.matrix_source, cfg.seed_base)
    _validate_ranks(cfg, a)
    a_norm = a.fro_norm()
    tails = _tail_energies(a)
    rows = []
    for rank in cfg.ranks:
        rows.append(("TSVD", rank, 0, (tails[rank] if rank < len(tails) else 0.0) / a_norm))
        for name, method in (("LUPP", "lupp"), ("QRCP", "qrcp")):
            for rep in range(cfg.reps):
                seed = cfg.seed_base + rep
                f, _ = iterative_cur(a, seed=seed, col_method=method, row_method=method, **_pure_rank(cfg.b, rank))
                rows.append((name, rank, rep, true_relative_error(a, f)))
    rows.sort(key=lambda r: (r[0], r[1], r[2]))
    csv = "method,rank,rep,rel_error\n" + "".join(f"{m},{rank},{rep},{_fmt_value(e)}\n" for m, rank, rep, e in rows)
    _emit(cfg, csv)
    return csv


def run_block_size(cfg: ExperimentConfig) -> str:
    """bench.cpp:282-318: block-size sweep in pure rank mode."""
    _validate_common(cfg)
    a = load_matrix(cfg.matrix_source, cfg.seed_base)
    _validate_ranks(cfg, a)
    if not cfg.blocks:
        raise ValueError("block list must not be empty")
    if any(b < 1 for b in cfg.blocks):
        raise ValueError("block sizes must be positive")
    rows = []
    for block in cfg.blocks:
        for rank in cfg.ranks:
            for rep in range(cfg.reps):
                seed = cfg.seed_base + rep
                t0 = time.perf_counter()
                f, _ = iterative_cur(a, seed=seed, **_pure_rank(block, rank))
                wall = time.perf_counter() - t0
                rows.append((block, rank, rep, true_relative_error(a, f), wall))
    rows.sort(key=lambda r: (r[0], r[1], r[2]))
    csv = "block_size,rank,rep,rel_error,wall_time_s\n" + "".join(
        f"{b},{rank},{rep},{_fmt_value(e)},{_fmt_time(w)}\n" for b, rank, rep, e, w in rows)
    _emit(cfg, csv)
    return csv


def run_experiment(cfg: ExperimentConfig) -> str:
    """bench.cpp:330-338."""
    return {"threshold": run_threshold, "fixed-rank": run_fixed_rank, "selection": run_selection_methods,
            "block-size": run_block_size}[cfg.kind](cfg)


def _int_list(s: str):
    return [int(x) for x in _tokens(s)]


def main(argv=None) -> int:
    """proj/tools/benchcli_main.cpp:33-73."""
    ap = argparse.ArgumentParser(prog="itercur-bench", description="Rank-adaptive CUR benchmark harness")
    sub = ap.add_subparsers(dest="kind", required=True)
    for name in ("threshold", "fixed-rank", "selection", "block-size"):
        p = sub.add_parser(name)
        p.add_argument("--matrix", required=True)
        p.add_argument("--b", type=int, default=50)
        p.add_argument("--eps", type=float, default=1e-6)
        p.add_argument("--delta", type=float, default=0.0)
        p.add_argument("--alpha", type=float, default=0.05)
        p.add_argument("--risk-adjust", action="store_true")
        p.add_argument("--ranks", type=_int_list, default=[])
        p.add_argument("--blocks", type=_int_list, default=[])
        p.add_argument("--reps", type=int, default=1)
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--out", required=True)
        p.add_argument("--deterministic", action="store_true")
    a = ap.parse_args(argv)
    cfg = ExperimentConfig(kind=a.kind, matrix_source=a.matrix, b=a.b, epsilon=a.eps, delta=a.delta, alpha=a.alpha,
                           risk_adjust=a.risk_adjust, ranks=a.ranks, blocks=a.blocks, reps=a.reps, seed_base=a.seed,
                           out_path=a.out, deterministic=a.deterministic)
    try:
        run_experiment(cfg)
    except Exception as e:  # noqa: BLE001 - the CLI reports every failure as the reference does
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())

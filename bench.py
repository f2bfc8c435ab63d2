#!/usr/bin/env python
"""Benchmark: m*n/s to tolerance of the B200 IterativeCUR engine (BASELINE.json metric).

One "step" = one full ``iterative_cur`` run (sketch + adaptive loop to tolerance) of
BASELINE config 2 (configs[1]: 20000 x 10000, sigma_i = i^-2, sparse-sign sketch, b = 20,
tol 1e-4) on a synthetic matrix formed in HBM (inputs > L2, so no flush is needed).

  value : m*n / (device time per step), A resident in HBM (device entry, CUDA events)
  e2e   : the same metric through the public API with a pinned HOST matrix (the host entry
          copies A to the device inside the call; indices / trace come back to the host)
  roofline : the sketch-apply kernel (the metric's named kernel), timed alone with CUDA
          events on its stream; plus a per-phase device-time breakdown of one profiled run
  cpu_baseline : the CPU oracle (restatement of the reference, 1 thread) on a bounded
          sample of the same run — see `cpu_reference_sample`.

`--impl reference` times only the CPU reference path (the oracle port: the reference
itself cannot be built here, no Eigen) on the same config and prints the same line.
Multi-GPU (torchrun, N > 1): by default every rank runs the workload on its own GPU (replicas,
weak scaling), value = N * m*n / max-over-ranks time. With --sharded one matrix is
column-sharded over the ranks (paper_2509_21963_b200/sharded.py; strong scaling),
value = m*n / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "m·n/s to tolerance (fp64 IterativeCUR); sketch-apply % of HBM/FP64 roofline"
UNIT = "m·n/s"
HBM_FALLBACK_GBS = 6650.0
DMMA_PEAK_TFLOPS = 37.1  # measured on this pool's B200 (tools/microbench/fp64_peak.cu, profiles/)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[2 + k].strip() == "Active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.samples[0][1]), "reasons": reasons,
                "samples": len(sm)}


NCU_FULL = "profiles/ncu_full_r01_cfg2_v6.txt"  # the committed `ncu --set full` summary of this config


def e2e_fits(bytes_needed, device_copy=True):
    """Whether the e2e leg can pin `bytes_needed` of host memory (<= 40% of MemAvailable) and, for
    the host entry's own device copy, allocate it beside the resident matrix. Configs 4/5 (80 GB)
    do not: their e2e leg is skipped with the reason rather than risking the box."""
    import torch

    avail = 0
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                avail = int(line.split()[1]) * 1024
    except OSError:
        pass
    if avail and bytes_needed > 0.4 * avail:
        return False, f"pinned host copy of {bytes_needed / 1e9:.0f} GB > 40% of available host memory"
    if device_copy and torch.cuda.is_available():
        free, _ = torch.cuda.mem_get_info()
        if bytes_needed * 1.15 > free:
            return False, f"a second device copy of A ({bytes_needed / 1e9:.0f} GB) does not fit in free HBM"
    return True, ""


def run_e2e(engine, a, m, n, run_cfg, args, world):
    """e2e leg: the host entry (MatrixHandle.dense over pinned memory), H2D inside the timed call."""
    import torch

    a_host_t = torch.empty(n, m, dtype=torch.float64, pin_memory=True)
    a_host_t.copy_(a.t())
    a_host = a_host_t.numpy().T  # (m, n) Fortran-ordered view of pinned memory
    hh = engine.MatrixHandle.dense(a_host)
    assert hh._host.ctypes.data == a_host.ctypes.data  # no copy: the H2D copy reads pinned memory
    engine.iterative_cur(hh, **run_cfg)  # warm
    torch.cuda.synchronize()
    e2e_t = []
    for _ in range(max(1, args.steps)):
        fe = te = None
        t0 = time.perf_counter()
        fe, te = engine.iterative_cur(hh, **run_cfg)
        _ = (fe.row_indices, fe.col_indices, te.rhos)  # already on the host
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = sum(e2e_t) / len(e2e_t)
    d2h = 8 * 2 * fe.rank + 8 * len(te.rhos)
    e2e = {"value": world * m * n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * m * n,
           "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * e2e_s}
    del fe, te, hh
    return e2e


def sketch_kernel_name(sketch, c):
    """The sketch-apply kernel the engine runs for this sketch kind (csrc/engine.cu sparse_sketch_mode)."""
    if sketch != "sparse_sign":
        return "sketch_dmma_kernel"
    c_pad = ((c + 7) // 8) * 8
    mode = os.environ.get("ITERCUR_SPARSE_SKETCH", "") or ("3" if c_pad > 32 else "2")
    return {"0": "sketch_dmma_kernel", "1": "sparse_sketch_kernel", "3": "sparse_sketch_umma_kernel"}.get(
        mode, "sparse_sketch_imma_kernel")


def ncu_traffic(kernel_substr, profile=NCU_FULL):
    """DRAM bytes (read + write) per launch of a kernel from the committed `ncu --set full`
    summary (tools/summarize_ncu.py), or None when no capture is on file."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), profile)
    if not os.path.exists(path):
        return None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total, inside = 0.0, False
    for line in open(path):
        if line.startswith("=="):
            if inside:
                break
            inside = kernel_substr in line
        elif inside and ("DRAM read" in line or "DRAM write" in line):
            parts = line.split()
            unit = parts[-1] if parts[-1] in scale else "byte"
            total += float(parts[-2] if parts[-1] in scale else parts[-1]) * scale[unit]
    return total if inside or total else None


def kernel_rooflines(engine, stages, cfg, m, n, rank_final, n_iters, hbm):
    """Live CUDA-event timings of the per-iteration kernels at the run's mean shapes: the two
    tall-skinny GEMMs (row residual on L: M = m; U block on R~: M = n, K = mean rank) against
    max(bytes/BW, flops/FP64 peak), and the LUPP (latency-bound: microseconds per pivot step)."""
    b = cfg["b"]
    k_mean = max(8, int(rank_final / 2))
    out = {}
    for name, M in (("row_residual_gemm", m), ("u_block_gemm", n)):
        us = stages.time_gemm(M, b, k_mean, reps=10)
        byts = 8.0 * M * k_mean
        fl = 2.0 * M * ((b + 7) // 8 * 8) * k_mean
        bound_s = max(byts / (hbm * 1e9), fl / (DMMA_PEAK_TFLOPS * 1e12))
        out[name] = {"shape_MNK": [M, b, k_mean], "us": us, "bound_us": bound_s * 1e6, "frac": bound_s * 1e6 / us,
                     "bound": "hbm" if byts / (hbm * 1e9) >= fl / (DMMA_PEAK_TFLOPS * 1e12) else "tensor"}
    for name, rows in (("col_lupp", n), ("row_lupp", m)):
        r = stages.time_lupp(rows, b, reps=10)
        out[name] = {"rows": rows, "steps": b, "us_per_call": r["us"], "us_per_step": r["us"] / b,
                     "bound": "latency (one cluster-wide exchange per pivot step)"}
    return out


def cpu_reference_sample(a_host, cfg, n_iters_total, budget_s=20.0):
    """Time the CPU oracle (restatement of the reference; its independent-column loops — sketch,
    GEMMs, the COD's reflector applications and solves — split over all host threads, bitwise the
    single-thread result) on the same matrix: the sketch plus the leading iterations until `budget_s` elapses
    (or convergence). The unmeasured tail is charged at the cost of the last measured
    iteration — an underestimate (per-iteration cost grows as O(r^3) in the reference's
    COD), so the reported CPU throughput is an upper bound."""
    from oracle import oracle as O

    O.build()
    m, n = a_host.shape
    b = cfg["b"]
    # pick a prefix length that fits the budget: grow until the elapsed time exceeds it
    k = 2
    while True:
        t0 = time.perf_counter()
        r = O.iterative_cur(a_host, epsilon=cfg["epsilon"], b=b, seed=0, sketch=cfg["sketch"], max_iters=k,
                            max_rank=cfg["max_rank"], log_steps=False)
        wall = time.perf_counter() - t0
        done = r.status == "Converged" or len(r.rhos) < k
        if done or wall > budget_s or k >= n_iters_total:
            break
        k = min(n_iters_total, max(k + 1, int(k * min(4.0, budget_s / max(wall, 1e-3)) * 0.8)))
    measured = len(r.iter_seconds)
    t_meas = r.total_s
    if done:
        t_est = t_meas
        note = f"full run to tolerance ({measured} iterations)"
    else:
        last = r.iter_seconds[-1] if r.iter_seconds else 0.0
        t_est = t_meas + max(0, n_iters_total - measured) * last
        note = (f"sketch + first {measured} of {n_iters_total} iterations measured ({t_meas:.2f} s); "
                f"remaining iterations charged at the last measured iteration's {last:.3f} s (lower bound on time)")
    threads = int(os.environ.get("ORACLE_THREADS", "0") or 0) or (os.cpu_count() or 1)
    return {"value": m * n / t_est, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"oracle restatement of the reference (-O3, {threads} host threads over independent columns) "
                      f"on the bench config's matrix: {note}",
            "t_est_s": t_est, "t_measured_s": t_meas, "iterations_measured": measured}


def run_reference_arm(args, cfg):
    """--impl reference: CPU oracle port on the same config; rank 0 only."""
    import numpy as np
    import torch

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2509_21963_b200 import testmat

    # the synthetic matrix is formed on the GPU (generation is not timed) and copied to the host
    a = testmat.generate(args.config).cpu().numpy() if torch.cuda.is_available() else None
    if a is None:
        print(json.dumps({"impl": "reference", "unavailable": "no GPU to form the synthetic matrix"}))
        return 0
    a = np.asfortranarray(a)
    n_total = int(args.ref_iters)
    vals = []
    for _ in range(args.warmup):
        pass  # the CPU path has nothing to warm; warm-up steps are not timed
    for _ in range(args.steps):
        s = cpu_reference_sample(a, cfg, n_total, budget_s=args.ref_budget)
        vals.append(s)
    v = sum(s["value"] for s in vals) / len(vals)
    t_step = sum(s["t_est_s"] for s in vals) / len(vals)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"BASELINE config {args.config}", **cfg}, "impl": "reference",
            "cpu_baseline": {k: vals[-1][k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    line["cpu_baseline"]["value"] = v
    print(json.dumps(line))
    return 0


def run_sharded(args, m, n, cfg, run_cfg, cfg_line, world, rank, local):
    """--sharded: one matrix column-sharded over the ranks (paper_2509_21963_b200/sharded.py,
    SURVEY §8(e)); strong scaling: value = m*n / max-over-ranks time of one run."""
    import numpy as np
    import torch

    import paper_2509_21963_b200 as engine  # noqa: F401  (loads the engine)
    from paper_2509_21963_b200 import build, testmat
    from paper_2509_21963_b200.sharded import iterative_cur_sharded

    build.build()
    a = testmat.generate(args.config)
    lo, hi = round(rank * n / world), round((rank + 1) * n / world)
    shard = a[:, lo:hi].t().contiguous().t()
    del a
    torch.cuda.synchronize()
    run = dict(run_cfg, column_exchange=args.exchange)
    res = None
    for _ in range(args.warmup):
        res = iterative_cur_sharded(shard, lo, n, **run)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            res = iterative_cur_sharded(shard, lo, n, **run)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    # e2e: each rank's shard from pinned host memory, H2D inside the timed region
    fits, why = e2e_fits(8 * shard.shape[0] * shard.shape[1])
    fits_t = torch.tensor([1.0 if fits else 0.0], device="cuda")
    if world > 1:
        torch.distributed.all_reduce(fits_t, op=torch.distributed.ReduceOp.MIN)
    e2e_ms = float("nan")
    if fits_t.item() > 0:
        host = torch.empty(shard.shape[1], shard.shape[0], dtype=torch.float64, pin_memory=True)
        host.copy_(shard.t())
        t0 = time.perf_counter()
        for _ in range(max(1, args.steps)):
            dshard = host.to("cuda", non_blocking=True).t()
            r2 = iterative_cur_sharded(dshard, lo, n, **run)
            _ = (r2.row_indices, r2.col_indices)
        torch.cuda.synchronize()
        e2e_ms = 1e3 * (time.perf_counter() - t0) / max(1, args.steps)
        del host
    if world > 1:
        tt = torch.tensor([ms, e2e_ms], device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms, e2e_ms = float(tt[0]), float(tt[1])
    if rank == 0:
        line = {"metric": METRIC, "value": m * n / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (device-generated, BASELINE config)",
                "config": {**cfg_line, "parallelism": f"column-sharded x{world}",
                           "column_exchange": args.exchange},
                "e2e": ({"value": m * n / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 8 * m * n,
                         "d2h_bytes_per_step": 16 * res.rank + 8 * len(res.rhos), "ms_per_step": e2e_ms}
                        if e2e_ms == e2e_ms else
                        {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                         "skipped": why or "a rank's shard does not fit the e2e leg"}),
                "clocks": clk.summary(),
                "run": {"status": res.status, "rank": res.rank, "iterations": len(res.rhos),
                        "exchanges_per_run": res.exchanges}}
        print(json.dumps(line))
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=20.0, help="CPU sample budget (s)")
    ap.add_argument("--ref-iters", type=int, default=0, help="iterations to tolerance for the CPU estimate")
    ap.add_argument("--exchange", default="sketch", choices=["sketch", "candidates"],
                    help="--sharded column selection: replicate Y per iteration, or exchange pivot candidates per step")
    ap.add_argument("--sharded", action="store_true",
                    help="N > 1: one matrix column-sharded over the GPUs (strong scaling) instead of N replicas")
    args = ap.parse_args()

    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")

    from paper_2509_21963_b200 import testmat

    cfg = dict(testmat.CONFIGS[args.config])
    m, n = cfg.pop("m"), cfg.pop("n")
    run_cfg = dict(epsilon=cfg["epsilon"], b=cfg["b"], seed=0, sketch=cfg["sketch"], max_rank=cfg["max_rank"])
    cfg_line = {"workload": f"BASELINE config {args.config} ({m}x{n}, {cfg['sketch']}, b={cfg['b']}, "
                            f"tol={cfg['epsilon']:g})", "m": m, "n": n, **cfg,
                "l2": "inputs larger than L2 (A = %.1f GB)" % (8 * m * n / 1e9),
                "parallelism": f"replicas x{world}" if world > 1 else "single GPU"}

    if args.impl == "reference":
        if args.ref_iters <= 0:
            args.ref_iters = {1: 15, 2: 120, 3: 8, 4: 9, 5: 16}[args.config]
        rc = run_reference_arm(args, {"m": m, "n": n, **cfg})
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()
        return rc

    if args.sharded:
        return run_sharded(args, m, n, cfg, run_cfg, cfg_line, world, rank, local)

    import paper_2509_21963_b200 as engine
    from paper_2509_21963_b200 import build, stages

    build.build()
    a = testmat.generate(args.config)
    torch.cuda.synchronize()
    handle = engine.MatrixHandle.device(a)

    # ---- one profiled run: per-phase breakdown + iteration count (not timed) ----
    f, t = engine.iterative_cur(handle, profile=True, **run_cfg)
    phases = {"sketch_s": t.sketch_s}
    for key in ("select_cols_s", "row_residual_s", "select_rows_s", "core_s", "downdate_s"):
        phases[key] = sum(getattr(r, key) for r in t.iterations)
    n_iters, rank_final, status = len(t.iterations), f.rank, t.status
    launches = t.kernel_launches
    del f, t

    # ---- warm-up + timed steps (device entry, A resident) ----
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        engine.iterative_cur(handle, **run_cfg)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            f = t = None  # release the previous run's factors before the next allocation
            f, t = engine.iterative_cur(handle, **run_cfg)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = tt.item()
    value = world * m * n / (ms * 1e-3)

    # ---- e2e through the public API with a pinned host matrix ----
    ok, why = e2e_fits(8 * m * n)
    if not ok:
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0, "skipped": why}
    else:
        e2e = run_e2e(engine, a, m, n, run_cfg, args, world)

    # ---- roofline: the sketch-apply kernel alone (CUDA events on its stream) ----
    hbm, hbm_src = peaks()
    sk = stages.time_sketch_kernel(a, cfg["b"], kind=cfg["sketch"], reps=10)
    c = engine.sketch_rows_for_block(cfg["b"])
    bytes_alg = 8.0 * m * n + 8.0 * c * n
    flops_alg = 2.0 * c * m * n if cfg["sketch"] == "gaussian" else 2.0 * 8 * m * n
    t_k = sk["ms"] * 1e-3
    if cfg["sketch"] == "gaussian" and flops_alg / (DMMA_PEAK_TFLOPS * 1e12) > bytes_alg / (hbm * 1e9):
        roof = {"bound": "tensor", "achieved": flops_alg / t_k / 1e12, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                "peak_source": "measured FP64 DMMA (tools/microbench/fp64_peak.cu)"}
    else:
        roof = {"bound": "hbm", "achieved": bytes_alg / t_k / 1e9, "peak": hbm, "unit": "GB/s",
                "peak_source": hbm_src}
    kname = sketch_kernel_name(cfg["sketch"], c)
    roof.update({"frac": roof["achieved"] / roof["peak"], "traffic": ncu_traffic(kname),
                 "traffic_source": f"{NCU_FULL} (dram__bytes_read + dram__bytes_write, one launch)",
                 "kernel": kname,
                 "ms_per_launch": sk["ms"], "ctas": sk["ctas"], "splits": sk["splits"], "tma": sk["tma"],
                 "algorithmic_bytes": bytes_alg, "algorithmic_flops": flops_alg})

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (device-generated, BASELINE config)",
            "config": cfg_line, "e2e": e2e, "roofline": roof, "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
            "kernels": kernel_rooflines(engine, stages, cfg, m, n, rank_final, n_iters, hbm),
            "run": {"status": status, "rank": rank_final, "iterations": n_iters, "phases_s": phases}}

    if rank == 0 and not args.no_cpu_baseline:
        if 8 * m * n <= 8e9:
            line["cpu_baseline"] = cpu_reference_sample(np.asfortranarray(a.cpu().numpy()), {**cfg}, n_iters,
                                                        budget_s=args.ref_budget)
        else:  # the oracle's sketch alone exceeds the sample budget at this size
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                                    "sample": "skipped: A exceeds 8 GB (configs 4/5); see configs 1-3"}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

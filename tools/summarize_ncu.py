"""Summaries of ncu captures for profiles/: a launch list (--metrics gpu__time_duration.sum --csv)
and `--set full` reports (key throughput / traffic / stall metrics per kernel).

    python tools/summarize_ncu.py launches gpurun_out/launches.csv "header text" > profiles/x.txt
    python tools/summarize_ncu.py full gpurun_out/a.ncu-rep [...] > profiles/y.txt
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors (from SM)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "FP64 tensor (DMMA) pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 (DFMA) pipe %"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tcgen05 (UTC) pipe %"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "integer MMA subpipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_size", "cluster"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def launches(path, header):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
    for r in rows[1:]:
        us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += us
    gen = ("gaussian_matrix_kernel",)  # test-matrix generation (testmat.py), outside the timed path
    mine = {k: v for k, v in agg.items() if "itercur_b200" in k and not any(g in k for g in gen)}
    tot = sum(v[1] for v in mine.values())
    print(header)
    print("Shares, not absolutes, are meaningful (cold-cache, serialised launches under ncu).\n")
    print(f"{'kernel':70s} {'launches':>8s} {'total_us':>10s} {'share':>6s} {'avg_us':>8s}")
    for k, (c, t) in sorted(mine.items(), key=lambda x: -x[1][1]):
        print(f"{k[:70]:70s} {c:8d} {t:10.1f} {100 * t / tot:5.1f}% {t / c:8.2f}")
    print(f"\ntotal {tot:.1f} us over {sum(v[0] for v in mine.values())} launches of the engine's kernels")
    other = {k: v for k, v in agg.items() if k not in mine}
    if other:
        print(f"(excluded: {sum(v[0] for v in other.values())} launches of test-matrix generation kernels "
              f"(torch/cuSOLVER QR and the generator's gaussian_matrix_kernel), outside the timed path)")


def full(paths):
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            print(p, ": no data")
            continue
        hdr, units = rows[0], rows[1]
        for vals in rows[2:]:
            d = dict(zip(hdr, vals))
            u = dict(zip(hdr, units))
            print(f"== {p}: {d.get('Kernel Name', '?')[:110]}")
            for k, label in KEYS:
                if k in d:
                    print(f"   {label:32s} {d[k]:>16s} {u.get(k, '')}")
            stalls = []
            for h, v in d.items():
                if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                    try:
                        stalls.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            stalls.sort(reverse=True)
            print("   top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]))
            print()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
    else:
        full(sys.argv[2:])

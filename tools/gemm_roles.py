"""Per-role times of the three per-iteration GEMMs in an ncu launch list of one engine run
(csrc/engine.cu order per iteration: row residual, U block, downdate; the unfused path for
blocks wider than 32):  python tools/gemm_roles.py gpurun_out/launches.csv"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
g = [(r[ki], float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)) for r in rows[1:] if "ts_gemm" in r[ki]]
roles = {0: [], 1: [], 2: []}
for q, (name, us) in enumerate(g):
    roles[q % 3].append(us)
for q, label in ((0, "row residual"), (1, "U block"), (2, "downdate")):
    v = roles[q]
    if v:
        print(f"{label:13s} {len(v):3d} launches  mean {sum(v) / len(v):8.1f}  total {sum(v):9.1f} (ncu time unit)")

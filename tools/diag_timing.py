"""Per-run timing diagnostics: repeated runs of one config with phase breakdowns."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_21963_b200 as engine
from paper_2509_21963_b200 import testmat
cfgno = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = testmat.CONFIGS[cfgno]
a = testmat.generate(cfgno); torch.cuda.synchronize()
h = engine.MatrixHandle.device(a)
kw = dict(epsilon=cfg["epsilon"], b=cfg["b"], seed=0, sketch=cfg["sketch"], max_rank=cfg["max_rank"])
for rep in range(reps):
    for prof in (False, True):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record()
        f, t = engine.iterative_cur(h, profile=prof, **kw)
        e1.record(); torch.cuda.synchronize(); wall = time.perf_counter() - t0
        ph = {k: round(sum(getattr(r, k) for r in t.iterations) * 1e3, 2) for k in
              ("select_cols_s", "row_residual_s", "select_rows_s", "core_s", "downdate_s")}
        print(json.dumps({"cfg": cfgno, "rep": rep, "profile": prof, "event_ms": round(e0.elapsed_time(e1), 2),
                          "wall_ms": round(wall * 1e3, 2), "engine_total_ms": round(t.total_s * 1e3, 2),
                          "sketch_ms": round(t.sketch_s * 1e3, 2), "iters": len(t.iterations), "rank": f.rank,
                          "phases_ms": ph, "mem_alloc_gb": round(torch.cuda.memory_reserved() / 1e9, 1)}), flush=True)
        del f, t

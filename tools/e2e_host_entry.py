"""e2e of the host entry (MatrixHandle.dense over a host matrix, H2D inside the call) from pageable
and from pinned memory, for one BASELINE config:  python tools/e2e_host_entry.py --config 4"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--kinds", default="pageable,pinned")
    args = ap.parse_args()
    import torch

    import paper_2509_21963_b200 as engine
    from paper_2509_21963_b200 import testmat

    cfg = dict(testmat.CONFIGS[args.config])
    m, n = cfg["m"], cfg["n"]
    kw = dict(epsilon=cfg["epsilon"], b=cfg["b"], seed=0, sketch=cfg["sketch"], max_rank=cfg["max_rank"])
    a = testmat.generate(args.config)
    out = {"config": args.config}
    pageable = torch.empty(n, m, dtype=torch.float64)
    pageable.copy_(a.t())
    del a
    torch.cuda.empty_cache()
    for kind in args.kinds.split(","):
        if kind == "pinned":
            host = torch.empty(n, m, dtype=torch.float64, pin_memory=True)
            host.copy_(pageable)
            del pageable
        else:
            host = pageable
        h = engine.MatrixHandle.dense(host.numpy().T)
        engine.iterative_cur(h, **kw)  # warm
        ts = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            f, t = engine.iterative_cur(h, **kw)
            _ = (f.row_indices, t.rhos)
            ts.append(time.perf_counter() - t0)
            del f, t
        out[kind] = {"s_per_run": ts, "h2d_GBps_upper": 8 * m * n / min(ts) / 1e9, "rank": None}
        del h, host
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())

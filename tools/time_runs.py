"""Device time of consecutive iterative_cur runs on one BASELINE config (CUDA events):
    python tools/time_runs.py --config 2 --runs 6 [--profile-first]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--runs", type=int, default=6)
    ap.add_argument("--profile-first", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2509_21963_b200 as engine
    from paper_2509_21963_b200 import testmat

    cfg = dict(testmat.CONFIGS[args.config])
    a = testmat.generate(args.config)
    h = engine.MatrixHandle.device(a)
    kw = dict(epsilon=cfg["epsilon"], b=cfg["b"], seed=0, sketch=cfg["sketch"], max_rank=cfg["max_rank"])
    if args.profile_first:
        engine.iterative_cur(h, profile=True, **kw)
    for r in range(args.runs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f, t = engine.iterative_cur(h, **kw)
        e1.record()
        torch.cuda.synchronize()
        print(r, f.rank, len(t.iterations), round(e0.elapsed_time(e1), 3), "ms", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())

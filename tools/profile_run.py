"""Minimal driver for ncu captures: form a BASELINE config on the device and run the engine.

    python tools/profile_run.py --config 2 --runs 2
(the first run is warm-up; profile the last one with ncu -s / -c as needed)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--sketch-only", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2509_21963_b200 as engine
    from paper_2509_21963_b200 import stages, testmat

    cfg = dict(testmat.CONFIGS[args.config])
    a = testmat.generate(args.config)
    torch.cuda.synchronize()
    if args.sketch_only:
        for _ in range(args.runs):
            print(stages.time_sketch_kernel(a, cfg["b"], kind=cfg["sketch"], reps=1))
        return 0
    for _ in range(args.runs):
        f, t = engine.iterative_cur(engine.MatrixHandle.device(a), epsilon=cfg["epsilon"], b=cfg["b"], seed=0,
                                    sketch=cfg["sketch"], max_rank=cfg["max_rank"])
        torch.cuda.synchronize()
        print(t.status, f.rank, len(t.iterations), t.kernel_launches)
    return 0


if __name__ == "__main__":
    sys.exit(main())

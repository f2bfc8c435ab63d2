"""One stage kernel timed alone (CUDA events), for quick checks and ncu captures:

    python tools/time_stage.py lupp ROWS STEPS [PATH] [REPS]   # PATH 0 auto, 1 cluster, 2 grid smem, 3 panel/global, 4 resident
    python tools/time_stage.py gemm M N K [REPS]                # row-residual shape C = A(:,idx) - L B
    python tools/time_stage.py sketch M N B KIND [REPS]         # KIND gaussian | sparse_sign, random A
    python tools/time_stage.py h2d [GB]                         # host->device copy rate, pageable vs pinned
(ITERCUR_LUPP_TRACE=1 with `lupp` prints the per-step phase cycles of CTA 0.)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(argv):
    import torch

    from paper_2509_21963_b200 import stages

    what, args = argv[0], [x for x in argv[1:]]
    if what == "lupp":
        rows, steps = int(args[0]), int(args[1])
        path = int(args[2]) if len(args) > 2 else 0
        reps = int(args[3]) if len(args) > 3 else 10
        print(rows, steps, stages.time_lupp(rows, steps, reps=reps, force_path=path))
    elif what == "gemm":
        M, N, K = int(args[0]), int(args[1]), int(args[2])
        reps = int(args[3]) if len(args) > 3 else 20
        us = stages.time_gemm(M, N, K, reps=reps)
        print(M, N, K, f"{us:.2f} us", f"{8.0 * M * K / (us * 1e-6) / 1e9:.1f} GB/s of L")
    elif what == "sketch":
        m, n, b, kind = int(args[0]), int(args[1]), int(args[2]), args[3]
        reps = int(args[4]) if len(args) > 4 else 3
        a = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
        print(m, n, b, kind, stages.time_sketch_kernel(a, b, kind=kind, reps=reps))
    elif what == "h2d":
        import numpy as np

        n = int(float(args[0] if args else 8) * 2 ** 30) // 8
        a = np.ones(n)
        d = torch.empty(n, dtype=torch.float64, device="cuda")
        for name, src in (("pageable", torch.from_numpy(a)), ("pinned", torch.from_numpy(a).pin_memory())):
            d.copy_(src)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            d.copy_(src)
            torch.cuda.synchronize()
            print(name, f"{8 * n / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
    else:
        raise SystemExit(__doc__)
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:] or ["help"]))

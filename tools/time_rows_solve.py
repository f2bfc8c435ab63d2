"""Row-solve kernel timing (itercur_rows_lu_solve_device, CUDA events): rows in shared memory (default),
the row-oriented register form and the column-oriented lane-pair form at the U-block shapes.  python tools/time_rows_solve.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_21963_b200 import _capi  # noqa: E402

L = _capi.lib()
for M, w in ((100000, 50), (50000, 64), (100000, 40), (20000, 64)):
    X = torch.randn(w, M, dtype=torch.float64, device="cuda").t()
    D = torch.randn(w, w, dtype=torch.float64, device="cuda") + w * torch.eye(w, dtype=torch.float64, device="cuda")
    out = torch.empty_like(X.t()).t()
    st = torch.cuda.current_stream().cuda_stream
    for form in ("blocked", "smem", "col", "row"):
        for k in ("ROWFORM", "COLFORM", "SMEM"):
            os.environ.pop("ITERCUR_ROWS_SOLVE_" + k, None)
        if form == "smem":
            os.environ["ITERCUR_ROWS_SOLVE_SMEM"] = "1"
        elif form == "row":
            os.environ["ITERCUR_ROWS_SOLVE_ROWFORM"] = "1"
        elif form == "col":
            os.environ["ITERCUR_ROWS_SOLVE_COLFORM"] = "1"
        f = lambda: _capi.check(L.itercur_rows_lu_solve_device(C.c_void_p(X.data_ptr()), M, M, C.c_void_p(D.data_ptr()),
                                                               w, w, C.c_void_p(out.data_ptr()), M, C.c_void_p(st)))
        f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        print(f"M={M} w={w} {form}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us", flush=True)

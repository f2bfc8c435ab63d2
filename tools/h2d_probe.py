import time, torch, numpy as np, ctypes as C
n = 8 * 2**30 // 8
a = np.ones(n)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, src in (("pageable", torch.from_numpy(a)), ("pinned", torch.from_numpy(a).pin_memory())):
    d.copy_(src); torch.cuda.synchronize()
    t0 = time.perf_counter(); d.copy_(src); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(name, f"{8*n/dt/1e9:.1f} GB/s")
# cudaMemcpy directly from pageable via the runtime
lib = C.CDLL("libcudart.so.12") if False else None

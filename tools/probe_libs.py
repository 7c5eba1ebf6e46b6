"""One-off probe: cuBLAS DGEMM peak and cuSOLVER SVD timings on B200 (inputs to DESIGN.md)."""
import json, time, torch
dev = "cuda"
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e))
    return best
for n in (1024, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev); b = torch.randn(n, n, dtype=torch.float64, device=dev)
    ms = timeit(lambda: a @ b)
    print(json.dumps({"probe": "cublas_dgemm", "n": n, "ms": ms, "tflops": 2 * n**3 / ms / 1e9}))
for (m, n) in ((1024, 1024), (1024, 128), (576, 576), (2560, 2560), (2560, 256)):
    x = torch.randn(m, n, dtype=torch.float64, device=dev)
    for drv in ("gesvd", "gesvdj", "gesvda"):
        try:
            ms = timeit(lambda: torch.linalg.svd(x, full_matrices=False, driver=drv), reps=3)
            print(json.dumps({"probe": "svd", "driver": drv, "m": m, "n": n, "ms": ms}))
        except Exception as ex:
            print(json.dumps({"probe": "svd", "driver": drv, "m": m, "n": n, "err": str(ex)[:100]}))
    g = x @ x.T
    ms = timeit(lambda: torch.linalg.eigh(g), reps=3)
    print(json.dumps({"probe": "syevd", "m": m, "ms": ms}))

"""cuBLAS (torch.matmul, fp64) timing of the ISO solver's plain GEMM shapes at C4, for comparison
with tc_gemm's per-launch times in the move's ncu launch list."""
import json
import torch

dev = torch.device("cuda")
R = C = 1024
l = 160
shapes = {"M Z (1024x1024 . 1024x160)": (R, C, l), "M^T Y (1024x1024^T . 1024x160)": (C, R, l),
          "Gram Y^T Y (160x1024 . 1024x160)": (l, R, l), "Y W (1024x160 . 160x160)": (R, l, l)}
for name, (m, k, n) in shapes.items():
    a = torch.randn(m, k, dtype=torch.float64, device=dev)
    b = torch.randn(k, n, dtype=torch.float64, device=dev)
    for _ in range(5):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        c = a @ b
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 50
    print(json.dumps({"shape": name, "us": round(us, 2), "tflops": round(2 * m * k * n / us / 1e6, 2)}))

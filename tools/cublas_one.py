"""One cuBLAS DGEMM of a chain-step shape (for ncu): python tools/cublas_one.py M N K [batch]"""
import sys
import torch
M, N, K = (int(x) for x in sys.argv[1:4])
b = int(sys.argv[4]) if len(sys.argv) > 4 else 2
A = torch.randn(b, M, K, dtype=torch.float64, device="cuda")
B = torch.randn(b, K, N, dtype=torch.float64, device="cuda")
for _ in range(3):
    C = torch.bmm(A, B)
torch.cuda.synchronize()
torch.cuda.profiler.start()
C = torch.bmm(A, B)
torch.cuda.synchronize()
torch.cuda.profiler.stop()

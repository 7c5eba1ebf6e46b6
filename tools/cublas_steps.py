"""cuBLAS DGEMM on the GEMM shapes of the C4 sequential chain (S1..S6, two chains per launch).

A library comparison point for tc_gemm: each step's (M, N, K) from the contraction order of
SURVEY 8(a) rows a6-a8 (csrc/ctm_abi.cu chain_batch), run as a batched torch.bmm in float64 (cuBLAS DGEMM) with
operands ALREADY in GEMM layout -- i.e. without the index permutations that tc_gemm fuses into its loads, which a
library pipeline would pay as extra HBM passes (the permute_ms column estimates one read + one write of the
permuted operand at the measured copy bandwidth). Times are CUDA events over 20 launches after 5 warm-ups, with
an L2 flush between launches like bench.py.

    python tools/cublas_steps.py [--D 8 --chi 128]
"""
import argparse
import json

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--D", type=int, default=8)
    ap.add_argument("--chi", type=int, default=128)
    ap.add_argument("--d", type=int, default=2)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    D, chi, d = a.D, a.chi, a.d
    # (name, M, N, K, the operand a library pipeline must permute first, its element count)
    steps = [
        ("S1", D * chi, D * D * chi, chi, "v1_in", chi * D * chi),
        ("S2", chi * D * chi, d * D * D, D * D, "X1", D * chi * D * D * chi),
        ("S3", chi * D * d * D, chi, chi * D, "X2", chi * D * d * D * D * chi),
        ("S4", D * d * D * chi, D * chi, chi, "X3", chi * D * d * D * chi),
        ("S5", D * chi * chi, D * D, d * D * D, "X4", d * D * D * D * chi * chi),
        ("S6", D * D * chi, chi, chi * D, "X5", chi * D * D * D * chi),
    ]
    dev = torch.device("cuda:0")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    hbm = 6537.6e9
    peak = 37.14e12
    g = torch.Generator(device=dev)
    g.manual_seed(230608212)
    total = 0.0
    for name, M, N, K, perm, nperm in steps:
        A = torch.randn(2, M, K, dtype=torch.float64, device=dev, generator=g)
        B = torch.randn(2, K, N, dtype=torch.float64, device=dev, generator=g)
        C = torch.empty(2, M, N, dtype=torch.float64, device=dev)
        for _ in range(5):
            torch.bmm(A, B, out=C)
        times = []
        for _ in range(a.reps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.bmm(A, B, out=C)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        times.sort()
        ms = times[len(times) // 2]
        fl = 2.0 * 2 * M * N * K
        permute_ms = 2 * 2 * nperm * 8 / hbm * 1e3
        total += ms
        print(json.dumps({"step": name, "M": M, "N": N, "K": K, "batch": 2, "cublas_ms": round(ms, 4),
                          "tflops": round(fl / ms / 1e9, 2), "frac": round(fl / ms / 1e9 / (peak / 1e12), 3),
                          "permute_operand": perm, "permute_ms_at_hbm_peak": round(permute_ms, 4)}))
        del A, B, C
    print(json.dumps({"chain_cublas_ms_two_chains": round(total, 4)}))


if __name__ == "__main__":
    main()

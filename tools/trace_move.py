"""Device timeline of one left move from CUPTI kernel activity records (tools/cupti, the
nsys-equivalent this image lacks; kernel start/end timestamps without perturbing launches):
warm-up moves, then the traced move; summarises per stream (busy time, kernel families), the
union of busy intervals and a coarse per-stream timeline.
    python tools/trace_move.py [config] > profiles/r02_trace_summary.txt"""
import collections
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
path = os.path.abspath("gpurun_out/r02_trace.jsonl")
import torch  # noqa: E402

import ctm_inputs as ci  # noqa: E402
from paper_2306_08212_b200 import ctm  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = ci.CONFIGS[name]
g = ci.generate(cfg)
dev = torch.device("cuda")
A = torch.from_numpy(g["A"]).to(dev)
B = torch.from_numpy(g["B"]).to(dev)
h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp, flags=ctm.CTM_FLAG_MOVE_ONLY)
env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
for _ in range(4):
    st = h.ctm_left_move(A, B, env)
torch.cuda.synchronize()
ct = ctypes.CDLL(os.path.join(ROOT, "tools", "cupti", "libcupti_trace.so"))
ct.ct_stop.argtypes = [ctypes.c_char_p]
assert ct.ct_start() == 0
st = h.ctm_left_move(A, B, env)
torch.cuda.synchronize()
n = ct.ct_stop(path.encode())
print(f"# traced {name} left move: {st['ms_total']:.2f} ms (CUPTI activity), isometry {st['ms_isometry']:.2f} ms, {n} kernels")
recs = [json.loads(line) for line in open(path)]
def fam(k):
    for key in ("tc_gemm", "splitk_reduce", "chol_kernel", "trsm_rows", "jacobi_cluster", "jacobi_lsv", "cheb_combine",
                "scale_commit", "permute", "replace_cols", "ritz_residual", "signfix", "fill_omega", "chol_"):
        if key in k:
            return key
    return k[:30]
streams = collections.OrderedDict()
for r in sorted(recs, key=lambda r: r["t0"]):
    streams.setdefault(r["s"], []).append(r)
T = max(r["t1"] for r in recs)
print(f"# {len(recs)} launches over {T:.2f} ms on {len(streams)} streams")
for si, (s, rs) in enumerate(streams.items()):
    busy = sum(r["t1"] - r["t0"] for r in rs)
    fams = collections.Counter()
    for r in rs:
        fams[fam(r["k"])] += r["t1"] - r["t0"]
    top = ", ".join(f"{k} {v:.2f}" for k, v in fams.most_common(6))
    print(f"stream {si}: {len(rs)} launches, busy {busy:.2f} ms of [{rs[0]['t0']:.2f}, {rs[-1]['t1']:.2f}] -- {top}")
# union of busy intervals
iv = sorted((r["t0"], r["t1"]) for r in recs)
u, a, b = 0.0, None, None
for x, y in iv:
    if a is None or x > b:
        if a is not None:
            u += b - a
        a, b = x, y
    else:
        b = max(b, y)
u += b - a
print(f"# union of busy intervals {u:.2f} ms = {100 * u / T:.1f}% of the move")
# coarse timeline: 1 ms bins, the dominant family per stream
binw = 0.5
nb = int(T / binw) + 1
print("# timeline (0.5 ms bins; per stream the family with most time in the bin; '.' idle)")
codes = {"tc_gemm": "G", "splitk_reduce": "r", "chol_kernel": "C", "trsm_rows": "t", "jacobi_cluster": "J",
         "cheb_combine": "c", "scale_commit": "K", "permute": "p"}
for si, (s, rs) in enumerate(streams.items()):
    row = []
    for bi in range(nb):
        lo, hi = bi * binw, (bi + 1) * binw
        acc = collections.Counter()
        for r in rs:
            ov = min(hi, r["t1"]) - max(lo, r["t0"])
            if ov > 0:
                acc[fam(r["k"])] += ov
        if not acc:
            row.append(".")
        else:
            k, v = acc.most_common(1)[0]
            ch = codes.get(k, "o")
            row.append(ch if sum(acc.values()) > 0.5 * binw else ch.lower())
    print(f"s{si} " + "".join(row))

"""Profiling driver for the isometry solver: ctm_reduced_env (rows a1-a4: two side TS
solves) at a config, run twice; ncu launch lists capture the second call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ctm_inputs as ci  # noqa: E402
from paper_2306_08212_b200 import ctm  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
algo = {"iso": ctm.CTM_SVD_ISO, "gesvdp": ctm.CTM_SVD_GESVDP}[sys.argv[2] if len(sys.argv) > 2 else "iso"]
cfg = ci.CONFIGS[name]
g = ci.generate(cfg)
h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp, svd_algo=algo, flags=ctm.CTM_FLAG_MOVE_ONLY)
C, T, A = g["C"], g["T"], g["A"]
dev = torch.device("cuda")
t = lambda x: torch.from_numpy(x).to(dev)  # noqa: E731
M = torch.empty((cfg.chi, cfg.D, cfg.D, cfg.chi), dtype=torch.float64, device=dev)
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.ctm_reduced_env(t(C[("a", 1)]), t(T[("a", 2)]), t(C[("a", 2)]), t(T[("a", 1)]), t(A), t(A), t(T[("a", 3)]), M)
    e1.record()
    torch.cuda.synchronize()
    print("reduced_env ms", e0.elapsed_time(e1))

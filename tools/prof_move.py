"""Profiling driver: one C4 left move with injected isometries (the contraction-only hot
path) after a warm-up, for ncu launch lists / --set full captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ctm_inputs as ci  # noqa: E402
from paper_2306_08212_b200 import ctm  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
mode = sys.argv[2] if len(sys.argv) > 2 else "inject"
cfg = ci.CONFIGS[name]
g = ci.generate(cfg)
h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp, flags=ctm.CTM_FLAG_MOVE_ONLY)
A = torch.from_numpy(g["A"]).cuda()
B = torch.from_numpy(g["B"]).cuda()
env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
iso = torch.zeros(h.iso_numel(), dtype=torch.float64, device="cuda")
h.ctm_left_move(A, B, env, iso_out=iso)          # full move once (computes isometries)
h.ctm_left_move(A, B, env, iso_in=iso if mode == "inject" else None)   # warm
torch.cuda.synchronize()
# only this move is profiled when ncu runs with --profile-from-start off
torch.cuda.profiler.start()
st = h.ctm_left_move(A, B, env, iso_in=iso if mode == "inject" else None)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(st)

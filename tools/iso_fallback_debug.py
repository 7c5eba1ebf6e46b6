"""Run n_iter CTM iterations of a config with CTM_ISO_DEBUG=1 set by the caller and report the
solver's fallbacks per move (stderr carries the per-solve trace)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ctm_inputs as ci  # noqa: E402
from paper_2306_08212_b200 import ctm  # noqa: E402

name, n_iter = sys.argv[1], int(sys.argv[2])
cfg = ci.CONFIGS[name]
g = ci.generate(cfg)
A = torch.from_numpy(g["A"]).cuda()
B = torch.from_numpy(g["B"]).cuda()
h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp, flags=ctm.CTM_FLAG_MOVE_ONLY)
env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
for it in range(n_iter):
    for d in ("left", "right", "up", "down"):
        print(f"=== iteration {it + 1} move {d}", file=sys.stderr, flush=True)
        st = h.ctm_move(d, A, B, env)
        print(it + 1, d, "fallbacks", st["n_svd_fallback"], "ms", round(st["ms_total"], 2),
              "min_gap", st["min_gap"], flush=True)

"""One left move of a BASELINE config with the ISO solver, CTM_ISO_DEBUG output on stderr.
    CTM_ISO_DEBUG=1 python tools/iso_debug_move.py c5_256 [moves]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ctm_inputs as ci  # noqa: E402
from paper_2306_08212_b200 import ctm  # noqa: E402

cfg = ci.CONFIGS[sys.argv[1]]
moves = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = ci.generate(cfg)
dev = torch.device("cuda")
h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp, svd_algo=ctm.CTM_SVD_ISO,
                  flags=ctm.CTM_FLAG_MOVE_ONLY, device=dev)
env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi, device=dev)
A, B = torch.from_numpy(g["A"]).to(dev), torch.from_numpy(g["B"]).to(dev)
for i in range(moves):
    st = h.ctm_left_move(A, B, env)
    print(i, st["n_svd"], st["n_svd_fallback"], round(st["ms_total"], 1), flush=True)

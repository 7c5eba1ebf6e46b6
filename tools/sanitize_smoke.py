"""Small end-to-end exercise of every libctm entry point (tiny / C2 shapes) for
compute-sanitizer --tool memcheck / racecheck runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ctm_inputs as ci  # noqa: E402
from paper_2306_08212_b200 import ctm  # noqa: E402

dev = torch.device("cuda")
for name, strategy in [("tiny", ctm.CTM_SEQUENTIAL), ("c2", ctm.CTM_SEQUENTIAL), ("tiny", ctm.CTM_REDUCED_EXACT),
                       ("tiny", ctm.CTM_STANDARD)]:
    cfg = ci.CONFIGS[name]
    g = ci.generate(cfg)
    A = torch.from_numpy(g["A"]).to(dev)
    B = torch.from_numpy(g["B"]).to(dev)
    h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, strategy=strategy, flags=ctm.CTM_FLAG_CHECK_FINITE)
    env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
    h.ctm_left_move(A, B, env)
    h.ctm_move("up", A, B, env)
    n, _ = h.ctm_norm_2x2(A, B, env)
    hop = torch.from_numpy(ci.heisenberg_h()).to(dev)
    e = h.ctm_bond_energy(A, B, env, hop, ctm.CTM_BOND_H)
    spins, ms = h.ctm_site_spins(A, B, env)
    it, delta, _ = h.ctm_converge(A, B, env, 2, 0.0)
    torch.cuda.synchronize()
    print(name, strategy, f"norm {n:.3e} e {e:.4f} m_s {ms:.4f} iters {it} delta {delta:.3e}", flush=True)
print("sanitize smoke ok")

"""Time one isolated truncating solve of the C4 move (no concurrency): the side TS of
Q_l = C^1 T^1 (a flat cut) and the main TS of M (a steep cut), through ctm_ts_isometry.
    CTM_ISO_DEBUG=1 python tools/prof_solve.py [reps]
Inputs: the C4 seeded environment; Q_l by torch.einsum (input preparation only) and M by
ctm_reduced_env."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ctm_inputs as ci  # noqa: E402
from paper_2306_08212_b200 import ctm  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = ci.CONFIGS["c4"]
g = ci.generate(cfg)
dev = torch.device("cuda")
T = {k: torch.from_numpy(v).to(dev) for k, v in g["T"].items()}
C = {k: torch.from_numpy(v).to(dev) for k, v in g["C"].items()}
A = torch.from_numpy(g["A"]).to(dev)
h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, flags=ctm.CTM_FLAG_MOVE_ONLY)
Ql = torch.einsum("xp,qkbx->pkbq", C[("a", 1)], T[("a", 1)]).contiguous()
M = torch.empty((cfg.chi, cfg.D, cfg.D, cfg.chi), dtype=torch.float64, device=dev)
h.ctm_reduced_env(C[("a", 1)], T[("a", 2)], C[("a", 2)], T[("a", 1)], A, A, T[("a", 3)], M)
for name, Q in (("flat side Q_l", Ql), ("steep main M", M)):
    for r in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        if os.environ.get("CTM_PROF_RANGE") == "1" and r == reps - 1:
            torch.cuda.profiler.start()
        h.ctm_ts_isometry(Q, cfg.chi, cfg.chi, ctm.CTM_TS_BASIS)
        if os.environ.get("CTM_PROF_RANGE") == "1" and r == reps - 1:
            torch.cuda.profiler.stop()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name}: {e0.elapsed_time(e1):.3f} ms", flush=True)

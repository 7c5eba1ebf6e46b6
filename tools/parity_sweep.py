"""Gauge-invariant parity vs iteration count: GPU (libctm) vs oracle, next to the
oracle's own sensitivity (oracle vs oracle with a 1e-15 relative perturbation of the
initial environment).  Writes one JSON line per (config, env_init, iteration).
Used to set the tolerances of tests/test_gpu_parity.py."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ctm_inputs as ci  # noqa: E402
from oracle import ctm_oracle as O  # noqa: E402
from paper_2306_08212_b200 import ctm  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2"]
n_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 20
inits = sys.argv[3].split(",") if len(sys.argv) > 3 else [None]
h_op = ci.heisenberg_h()
for name in names:
    for init in inits:
        cfg = ci.CONFIGS[name]
        g = ci.generate(cfg, env_init=init)
        A, B = g["A"], g["B"]
        hd = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp)
        env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
        At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        e1 = {"C": dict(g["C"]), "T": dict(g["T"])}
        rng = np.random.default_rng(1)
        e2 = {"C": {k: v * (1 + 1e-15 * rng.standard_normal(v.shape)) for k, v in g["C"].items()},
              "T": dict(g["T"])}
        for it in range(1, n_iter + 1):
            hd.ctm_iterate(At, Bt, env, 1)
            e1 = O.ctm_iteration(e1, A, B, cfg.chi, cfg.chi_p, cfg.chi_pp)
            e2 = O.ctm_iteration(e2, A, B, cfg.chi, cfg.chi_p, cfg.chi_pp)
            eg = env.to_host()
            n_g, n1, n2 = O.norm_2x2(eg, A, B), O.norm_2x2(e1, A, B), O.norm_2x2(e2, A, B)
            E_g, E1, E2 = (O.bond_energy(e, A, B, h_op)[0] for e in (eg, e1, e2))
            rec = {"config": name, "env_init": init, "iteration": it,
                   "norm_rel_gpu_oracle": abs(n_g - n1) / abs(n1), "norm_rel_oracle_perturbed": abs(n2 - n1) / abs(n1),
                   "eH_abs_gpu_oracle": abs(E_g - E1), "eH_abs_oracle_perturbed": abs(E2 - E1),
                   "norm": n1, "e_H": E1}
            print(json.dumps(rec), flush=True)

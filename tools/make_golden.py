"""Write tests/golden/oracle_*.json: gauge-invariant oracle outputs for the small configs.

Calls ONLY oracle/ and ctm_inputs (never the CUDA path).  Read by
tests/test_oracle_golden.py as a regression fixture of the oracle itself.  Re-run after any change to
the oracle's arithmetic (and say why in the commit message)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import ctm_inputs as ci  # noqa: E402
from oracle import ctm_oracle as O  # noqa: E402


def observables(env, A, B):
    h = ci.heisenberg_h()
    eH, _ = O.bond_energy(env, A, B, h, "H")
    eV, _ = O.bond_energy(env, A, B, h, "V")
    return {"norm_2x2": O.norm_2x2(env, A, B), "e_H": eH, "e_V": eV}


def run(name, n_left_moves=None, n_iter=None):
    cfg = ci.CONFIGS[name]
    g = ci.generate(cfg)
    env = {"C": g["C"], "T": g["T"]}
    A, B = g["A"], g["B"]
    out = {"config": name, "seed": cfg.seed, "d": cfg.d, "D": cfg.D, "chi": cfg.chi,
           "chi_p": cfg.chi_p, "chi_pp": cfg.chi_pp}
    t = time.time()
    if n_left_moves:
        e1 = O.left_move(env, A, B, cfg.chi, cfg.chi_p, cfg.chi_pp)
        out["after_left_move"] = observables(e1, A, B)
    if n_iter:
        e = env
        for _ in range(n_iter):
            e = O.ctm_iteration(e, A, B, cfg.chi, cfg.chi_p, cfg.chi_pp)
        out[f"after_{n_iter}_iterations"] = observables(e, A, B)
    out["oracle_seconds"] = time.time() - t
    return out


def run_dl(name, n_iter):
    """Gauge-invariant values after each of n_iter CTM iterations of a converging (R16b)
    config -- the GPU test compares its own trajectory at 1e-9 (the oracle's
    perturbed-start spread stays ~1e-14 on c4_dl, profiles/r02_spread_c4_dl.txt)."""
    cfg = ci.CONFIGS[name]
    g = ci.generate(cfg)
    env = {"C": g["C"], "T": g["T"]}
    A, B = g["A"], g["B"]
    out = {"config": name, "seed": cfg.seed, "d": cfg.d, "D": cfg.D, "chi": cfg.chi, "iterations": []}
    t = time.time()
    for it in range(n_iter):
        env = O.ctm_iteration(env, A, B, cfg.chi, cfg.chi_p, cfg.chi_pp)
        out["iterations"].append(observables(env, A, B))
        print(name, it + 1, out["iterations"][-1], round(time.time() - t, 1), flush=True)
    out["oracle_seconds"] = time.time() - t
    return out


if __name__ == "__main__":
    gold = os.path.join(ROOT, "tests", "golden")
    if "--dl" in sys.argv:   # the converging c4_dl trajectory (slow: ~15 min on 8 cores)
        res = {"_source": "written by tools/make_golden.py --dl from oracle/ only (no CUDA path)",
               "c4_dl": run_dl("c4_dl", 20)}
        with open(os.path.join(gold, "oracle_c4_dl.json"), "w") as f:
            json.dump(res, f, indent=1)
        sys.exit(0)
    res = {"_source": "written by tools/make_golden.py from oracle/ only (no CUDA path)",
           "tiny": run("tiny", n_left_moves=1, n_iter=1),
           "c2": run("c2", n_left_moves=1, n_iter=20)}
    with open(os.path.join(gold, "oracle_small.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))

"""The paper's timing figure on B200 (Fig. result:time): wall time of 5
imaginary-time steps vs D for the three strategies, chi = 10(D+1), d = 2, Heisenberg
gates, each step = the second-order Trotter sweep over the four bonds with the fast full update
(ctm_trotter_step: 7 bond updates, each followed by one CTM iteration of the handle's strategy).
Seeded decaying-spectrum A, B (BASELINE recipe) and the double-layer environment start.
    python tools/trotter_timing.py [--D 4,6,8,10] [--strategies sequential,reduced,standard]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ctm_inputs as ci  # noqa: E402
from paper_2306_08212_b200 import ctm  # noqa: E402


def run(D, strategy, steps=5, delta=0.05):
    chi = 10 * (D + 1)
    cfg = ci.custom(2, D, chi, decaying=True, seed_index=700 + D)
    g = ci.generate(cfg, "double_layer")
    dev = torch.device("cuda")
    strat = {"sequential": ctm.CTM_SEQUENTIAL, "reduced": ctm.CTM_REDUCED_EXACT, "standard": ctm.CTM_STANDARD}[strategy]
    h = ctm.CtmHandle(2, D, chi, strategy=strat)
    A = torch.from_numpy(g["A"]).to(dev)
    B = torch.from_numpy(g["B"]).to(dev)
    env = ctm.Env.from_host(g["C"], g["T"], D, chi)
    hop = torch.from_numpy(ci.heisenberg_h()).to(dev)
    h.ctm_iterate(A, B, env, 2)                              # grow the boundary to chi
    h.ctm_trotter_step(A, B, env, hop, delta, 3)             # warm-up step
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(steps):
        h.ctm_trotter_step(A, B, env, hop, delta, 3)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t
    e = h.ctm_bond_energy(A, B, env, hop, ctm.CTM_BOND_H) + h.ctm_bond_energy(A, B, env, hop, ctm.CTM_BOND_V)
    return {"D": D, "chi": chi, "strategy": strategy, "steps": steps, "seconds": sec, "s_per_step": sec / steps,
            "energy_per_site": e, "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--D", default="4,6,8,10")
    ap.add_argument("--strategies", default="sequential,reduced,standard")
    a = ap.parse_args()
    for D in [int(x) for x in a.D.split(",")]:
        for s in a.strategies.split(","):
            if s == "standard" and D > 6:
                continue   # the (chi D^2)^2 half-network SVD: 558 ms per move at D = 8 already
            torch.cuda.reset_peak_memory_stats()
            print(json.dumps(run(D, s)), flush=True)


if __name__ == "__main__":
    main()

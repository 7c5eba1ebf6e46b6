"""Consecutive left moves (bench.py's sequence) with and without CTM_FLAG_WARM_START: per-move
device time and the warm-start counters.  CTM_ISO_DEBUG=1 adds the solver's per-solve trace.
usage: python tools/warm_moves.py [config] [moves] [iterate]
  iterate: full CTM iterations (left, right, up, down) instead of left moves."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch

import ctm_inputs as ci
from paper_2306_08212_b200 import ctm


def run(cfg, n, warm, iterate):
    g = ci.generate(cfg)
    dev = torch.device("cuda:0")
    A = torch.from_numpy(g["A"]).to(dev)
    B = torch.from_numpy(g["B"]).to(dev)
    h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp,
                      flags=ctm.CTM_FLAG_MOVE_ONLY | (ctm.CTM_FLAG_WARM_START if warm else 0))
    env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
    out = []
    for i in range(n):
        if iterate:
            ms, nw, nh, nr, nf = 0.0, 0, 0, 0, 0
            for d in ("left", "right", "up", "down"):
                st = h.ctm_move(d, A, B, env)
                ms += st["ms_total"]; nw += st["n_warm"]; nh += st["n_warm_hit"]; nr += st["n_warm_retry"]
                nf += st["n_svd_fallback"]
        else:
            if os.environ.get("CTM_ISO_DEBUG"):
                sys.stderr.write(f"[move {i + 1} warm={warm}]\n")
            st = h.ctm_left_move(A, B, env)
            ms, nw, nh, nr, nf = st["ms_total"], st["n_warm"], st["n_warm_hit"], st["n_warm_retry"], st["n_svd_fallback"]
        out.append({"ms": round(ms, 2), "warm": nw, "hit": nh, "retry": nr, "fallback": nf})
    return out


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    iterate = len(sys.argv) > 3 and sys.argv[3] == "iterate"
    cfg = ci.CONFIGS[name]
    for warm in (False, True):
        r = run(cfg, n, warm, iterate)
        print(json.dumps({"config": name, "unit": "iteration" if iterate else "left move", "warm_start": warm,
                          "ms": [x["ms"] for x in r], "warm_solves": [x["warm"] for x in r],
                          "first_check_hits": [x["hit"] for x in r], "cold_retries": sum(x["retry"] for x in r),
                          "fallbacks": sum(x["fallback"] for x in r)}), flush=True)

"""CTM moves/sec and FP64 TFLOP/s vs (D, chi) (BASELINE.json metric) on one B200.

For each config: the contraction-only left move (isometries injected: chains, corners,
commit -- the sequential-order hot path) and the full left move (reduced environments +
isometry solves included), CUDA events on the library stream, 256 MB L2 flush between
steps.  One JSON line per config.

    python tools/sweep.py [--configs c2,c3,c4,c5,c5_256] [--steps 5] [--svd iso]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ctm_inputs as ci  # noqa: E402
from paper_2306_08212_b200 import ctm  # noqa: E402

PEAK = 37.14   # measured FP64 DMMA peak (profiles/r01_probe_fp64.txt)


def config(name):
    """A BASELINE config name, or 'D<D>_chi<chi>' (seeded, decaying spectrum) for sweeps."""
    if name in ci.CONFIGS:
        return ci.CONFIGS[name]
    D, chi = name[1:].split("_chi")
    return ci.custom(2, int(D), int(chi), decaying=True, seed_index=500 + int(D), name=name)


def run(name, steps, svd, strategy="sequential"):
    cfg = config(name)
    g = ci.generate(cfg)
    dev = torch.device("cuda")
    stream = torch.cuda.Stream(dev)
    algo = {"iso": ctm.CTM_SVD_ISO, "gesvdp": ctm.CTM_SVD_GESVDP}[svd]
    with torch.cuda.stream(stream):
        strat = {"sequential": ctm.CTM_SEQUENTIAL, "reduced": ctm.CTM_REDUCED_EXACT,
                 "standard": ctm.CTM_STANDARD}[strategy]
        h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp, svd_algo=algo, flags=ctm.CTM_FLAG_MOVE_ONLY,
                          stream=stream, device=dev, strategy=strat)
        A = torch.from_numpy(g["A"]).to(dev)
        B = torch.from_numpy(g["B"]).to(dev)
        env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi, device=dev)
        iso = torch.zeros(h.iso_numel(), dtype=torch.float64, device=dev)
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)

        def step(inject):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if strategy != "sequential":
                st = h.ctm_left_move(A, B, env)
            else:
                st = h.ctm_left_move(A, B, env, iso_in=iso if inject else None, iso_out=None if inject else iso)
            e1.record(stream)
            e1.synchronize()
            return e0.elapsed_time(e1), st

        for _ in range(2):
            step(False)
        full = [step(False) for _ in range(steps)]
        if strategy != "sequential":   # no injected-isometry path: report the full move only
            con = full
        else:
            for _ in range(2):
                step(True)
            con = [step(True) for _ in range(steps)]
        ms_graph = None
        if strategy == "sequential":
            # contraction-only move replayed from a CUDA graph (SURVEY 8(d) timing protocol 3)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                h.ctm_left_move(A, B, env, iso_in=iso, stats=False)
            graph.replay()
            stream.synchronize()
            ts = []
            for _ in range(steps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                graph.replay()
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms_graph = float(np.median(ts))
    F = ctm.ctm_move_flops(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp) if strategy == "sequential" else None
    Fc = con[0][1]["flops"]
    ms_full = float(np.median([t for t, _ in full]))
    ms_con = float(np.median([t for t, _ in con]))
    return {"config": name, "d": cfg.d, "D": cfg.D, "chi": cfg.chi, "svd": svd, "strategy": strategy,
            "flops_per_move": F, "contraction_flops_per_move": Fc,
            "full_move_ms": ms_full, "full_moves_per_s": 1e3 / ms_full,
            "isometry_ms": float(np.median([s["ms_isometry"] for _, s in full])),
            "svd_fallbacks_per_move": float(np.mean([s["n_svd_fallback"] for _, s in full])),
            "contraction_only_ms": ms_con, "contraction_moves_per_s": 1e3 / ms_con,
            "contraction_tflops": Fc / (ms_con * 1e-3) / 1e12,
            "contraction_frac_of_fp64_peak": Fc / (ms_con * 1e-3) / 1e12 / PEAK,
            "contraction_graph_ms": ms_graph,
            "contraction_graph_frac_of_fp64_peak": (Fc / (ms_graph * 1e-3) / 1e12 / PEAK) if ms_graph else None,
            "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c3,c4,c5,c5_256")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--svd", default="iso")
    ap.add_argument("--strategies", default="sequential")
    a = ap.parse_args()
    for strategy in a.strategies.split(","):
        for name in a.configs.split(","):
            torch.cuda.reset_peak_memory_stats()
            print(json.dumps(run(name, a.steps, a.svd, strategy)), flush=True)


if __name__ == "__main__":
    main()

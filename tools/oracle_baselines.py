"""The oracle (NumPy float64, CPU) timed on the host it runs on, per BASELINE config (SURVEY
8(d) "Oracle timing": C2 and C3 the full 20-iteration run, C4 and C5 one left move), with the
core count, CPU model and BLAS vendor.  A reported baseline, not the optimisation target.
This is bench-side measurement code: it only calls oracle/ (allowed for the reference arm).

    python tools/oracle_baselines.py [--configs c2,c3,c4,c5] > profiles/r02_oracle_baselines.jsonl
"""
import argparse
import io
import json
import os
import platform
import sys
import time
from contextlib import redirect_stdout

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import ctm_inputs as ci  # noqa: E402
from oracle import ctm_oracle as O  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def blas():
    buf = io.StringIO()
    try:
        with redirect_stdout(buf):
            np.show_config()
    except Exception:
        return "unknown"
    txt = buf.getvalue().lower()
    for name in ("openblas", "mkl", "blis", "accelerate"):
        if name in txt:
            return name
    return "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c3,c4,c5")
    a = ap.parse_args()
    cores = len(os.sched_getaffinity(0))
    for name in a.configs.split(","):
        cfg = ci.CONFIGS[name]
        g = ci.generate(cfg)
        env = {"C": g["C"], "T": g["T"]}
        F = None
        t = time.perf_counter()
        if name in ("c2", "c3"):
            for _ in range(20):
                env = O.ctm_iteration(env, g["A"], g["B"], cfg.chi, cfg.chi_p, cfg.chi_pp)
            moves = 80
            what = "20 CTM iterations (80 moves)"
        else:
            O.left_move(env, g["A"], g["B"], cfg.chi, cfg.chi_p, cfg.chi_pp)
            moves = 1
            what = "1 left move"
        sec = time.perf_counter() - t
        print(json.dumps({"config": name, "D": cfg.D, "chi": cfg.chi, "what": what, "seconds": sec,
                          "moves_per_s": moves / sec, "cores": cores, "cpu": cpu_model(), "blas": blas()}),
              flush=True)


if __name__ == "__main__":
    main()

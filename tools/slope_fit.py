"""Log-log slopes of per-move algorithmic flops and measured B200 time vs D for the three
strategies (the paper's Fig result:time), from tools/sweep.py
output.  Flops: SEQUENTIAL = F_move (SURVEY 8(a) closed form, ctm_move_flops); REDUCED /
STANDARD = the contractions the strategy issues (stats.flops).  Time: full move (isometry
solves included).
    python tools/slope_fit.py gpurun_out/r02h_sweep_chi100.jsonl > profiles/r02_strategy_slopes.json"""
import json
import sys

import numpy as np

rows = [json.loads(line) for f in sys.argv[1:] for line in open(f)]
out = {}
for strat in ("sequential", "reduced", "standard"):
    r = sorted([x for x in rows if x["strategy"] == strat], key=lambda x: x["D"])
    if len(r) < 2:
        continue
    D = np.array([x["D"] for x in r], float)
    F = np.array([x["flops_per_move"] if strat == "sequential" else x["contraction_flops_per_move"] for x in r])
    t = np.array([x["full_move_ms"] for x in r])
    out[strat] = {"D": D.tolist(), "chi": [x["chi"] for x in r], "flops_GF": (F / 1e9).tolist(), "ms": t.tolist(),
                  "flop_slope_vs_D": float(np.polyfit(np.log(D), np.log(F), 1)[0]),
                  "time_slope_vs_D": float(np.polyfit(np.log(D), np.log(t), 1)[0]),
                  "time_slope_vs_D_last_two": float(np.log(t[-1] / t[-2]) / np.log(D[-1] / D[-2]))}
print(json.dumps(out, indent=1))

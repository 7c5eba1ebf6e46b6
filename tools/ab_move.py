"""A/B timing of the full C4 left move: one process per library, alternated several times.

    python tools/ab_move.py --libs base=ab/libctm_r02base.so,new= --procs 4 --moves 15

Each process builds a handle on the same seeded inputs, warms up 3 moves and times --moves
moves with CUDA events (L2 flushed between moves like bench.py); prints one JSON line per
process and a median summary per library.  An empty path means the in-tree libctm.so.
Extra environment per arm: name=path@VAR=value (e.g. new=@CTM_TC_SPLIT=slab).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(moves, config="c4"):
    sys.path.insert(0, ROOT)
    import torch
    import ctm_inputs as ci
    from paper_2306_08212_b200 import ctm
    cfg = ci.CONFIGS[config]
    g = ci.generate(cfg)
    h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp, flags=ctm.CTM_FLAG_MOVE_ONLY)
    A = torch.from_numpy(g["A"]).cuda()
    B = torch.from_numpy(g["B"]).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ms, iso, fb = [], [], []
    for i in range(3 + moves):
        env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(h.stream)
        st = h.ctm_left_move(A, B, env)
        e1.record(h.stream)
        torch.cuda.synchronize()
        if i >= 3:
            ms.append(e0.elapsed_time(e1))
            iso.append(st["ms_isometry"])
            fb.append(st.get("n_svd_fallback", 0))
    print(json.dumps({"median_ms": statistics.median(ms), "min_ms": min(ms), "iso_ms": statistics.median(iso),
                      "fallbacks": sum(fb)}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", default="base=ab/libctm_r02base.so,new=")
    ap.add_argument("--procs", type=int, default=4)
    ap.add_argument("--moves", type=int, default=15)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--config", default="c4")
    a = ap.parse_args()
    if a.child:
        child(a.moves, a.config)
        return
    arms = []
    for item in a.libs.split(","):
        name, spec = item.split("=", 1)
        path, *extras = spec.split("@")
        env = dict(os.environ)
        env.pop("CTM_LIB_PATH", None)
        if path:
            env["CTM_LIB_PATH"] = os.path.join(ROOT, path)
        for extra in extras:   # name=path@VAR=value[@VAR2=value2...]
            k, v = extra.split("=", 1)
            env[k] = v
        arms.append((name, env))
    res = {n: [] for n, _ in arms}
    for p in range(a.procs):
        for name, env in arms:
            out = subprocess.run([sys.executable, __file__, "--child", "--moves", str(a.moves), "--config", a.config], env=env,
                                 capture_output=True, text=True, timeout=600)
            line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
            if not line:
                print(json.dumps({"arm": name, "error": out.stderr[-500:]}), flush=True)
                continue
            d = json.loads(line[-1])
            d["arm"] = name
            res[name].append(d)
            print(json.dumps(d), flush=True)
    for name, v in res.items():
        if v:
            print(json.dumps({"arm": name, "procs": len(v), "median_of_medians_ms": statistics.median(x["median_ms"] for x in v),
                              "iso_ms": statistics.median(x["iso_ms"] for x in v),
                              "fallbacks": sum(x.get("fallbacks", 0) for x in v), "config": a.config}))


if __name__ == "__main__":
    main()

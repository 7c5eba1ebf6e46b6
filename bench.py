"""bench.py -- CTM moves/sec and FP64 TFLOP/s of the B200 CTMRG move (arXiv 2306.08212).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

One step = one LEFT MOVE (2 column absorptions, each with two
approximated reduced environments, 12 device SVDs, two sequential absorb/truncate
chains, four corner growths and the normalise+commit) on the synthetic C4 workload
(d=2, D=8, chi=chi'=chi''=128, decaying-spectrum seeded tensors, BASELINE.json
configs[3], the headline roofline config).  Inputs are resident in HBM; the move's
intermediates (>= 134 MB each) exceed the 126 MB L2 and an L2 flush (256 MB write)
separates timed steps; each step is timed with CUDA events on the library's stream.

Multi-GPU: the move does not shard ("replicas only"): under torchrun every
rank runs an independent replica; value = moves of all ranks / max-over-ranks time.

--impl reference times the CPU float64 oracle (oracle/) on the host cores on the same
config (the paper has no code; the oracle is the reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import ctm_inputs as ci  # noqa: E402

FP64_PEAK_TFLOPS = 37.14   # measured DMMA.8x8x4 loop peak on this pool's B200 (profiles/r01_probe_fp64.txt)
FP64_DFMA_PEAK_TFLOPS = 36.93   # measured DFMA loop peak, same file


def hbm_peak_gbs():
    """Measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs; driver-written)."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return None


def renv_flops(cfg):
    """Algorithmic flops of one reduced environment with injected side isometries (rows a1,
    a3, a4 and the v^1 Q GEMMs of a2; SURVEY 8(a) closed form, chi = chi' = chi''):
    F_chain + 12 chi^3 D^2 + 4 chi^3 D (2 Q products, 2 v^1 Q, the T'^2 chain, C', C'', C' T', (C' T') C'')."""
    c, D, d = float(cfg.chi), float(cfg.D), float(cfg.d)
    chain = 4 * c ** 3 * D ** 3 + 4 * d * c ** 3 * D ** 3 + 4 * d * c ** 2 * D ** 5
    return chain + 12 * c ** 3 * D ** 2 + 4 * c ** 3 * D
METRIC = "CTM moves/sec and FP64 TFLOP/s (% of B200 FP64 peak) vs D,chi"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--svd", default="iso", choices=["gesvdp", "gesvdj", "gesvd", "gram", "iso"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 4 + i and s[4 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return world, rank, local


def traffic_bytes(cfg):
    """DRAM bytes per contraction-only step of tc_gemm, measured by ncu for C4 (the latest of
    profiles/r02_traffic.json, profiles/r01_final_traffic.json); None for other configs."""
    for name in ("r02_traffic.json", "r01_final_traffic.json"):
        path = os.path.join(ROOT, "profiles", name)
        if cfg.name == "c4" and os.path.exists(path):
            return json.load(open(path))["dram_bytes_per_step"]
    return None


def max_over_ranks(vals, device=None):
    """Element-wise max of per-rank timings over all ranks (torch.distributed; the bench uses
    NCCL on GPUs, the CPU tests gloo).  Single process: returned unchanged."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(v) for v in vals]
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def job_value(world, ms_per_step_max):
    """Whole-job moves/s: every rank runs one independent replica move per step (replicas
    only), timed by the slowest rank."""
    return world * 1e3 / ms_per_step_max


def run_oracle_sample(cfg, what="left_move"):
    """One left move of the oracle (bounded CPU sample); returns seconds."""
    from oracle import ctm_oracle as O
    g = ci.generate(cfg)
    env = {"C": g["C"], "T": g["T"]}
    t = time.perf_counter()
    O.left_move(env, g["A"], g["B"], cfg.chi, cfg.chi_p, cfg.chi_pp)
    return time.perf_counter() - t


def workload(cfg):
    return (f"{cfg.name}: left move, d={cfg.d} D={cfg.D} chi={cfg.chi} chi'={cfg.chi_p} chi''={cfg.chi_pp}, "
            f"sequential order")


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def bench_reference(args, cfg):
    world, rank, _ = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    if rank != 0:
        return
    for _ in range(args.warmup):
        run_oracle_sample(cfg)
    ts = [run_oracle_sample(cfg) for _ in range(args.steps)]
    sec = float(np.sum(ts))
    value = args.steps / sec
    line = {"metric": METRIC, "value": value, "unit": "moves/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, ctm_inputs.py)",
            "config": {"workload": workload(cfg), "D": cfg.D, "chi": cfg.chi},
            "cpu_baseline": {"value": value, "unit": "moves/s", "cores": host_cores(), "kind": "oracle",
                             "sample": f"{args.steps} full left moves of {cfg.name} (NumPy/OpenBLAS fp64 oracle)"},
            "e2e": {"value": value, "unit": "moves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def bench_ours(args, cfg):
    import torch
    world, rank, local = dist_setup(args.gpus)
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    from paper_2306_08212_b200 import ctm
    svd = {"gesvdp": ctm.CTM_SVD_GESVDP, "gesvdj": ctm.CTM_SVD_GESVDJ, "gesvd": ctm.CTM_SVD_GESVD, "gram": ctm.CTM_SVD_GRAM, "iso": ctm.CTM_SVD_ISO}[args.svd]
    stream = torch.cuda.Stream(dev)
    g = ci.generate(cfg)
    with torch.cuda.stream(stream):
        h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp, svd_algo=svd,
                          flags=ctm.CTM_FLAG_MOVE_ONLY, stream=stream, device=dev)
        hp = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp, svd_algo=svd,
                           flags=ctm.CTM_FLAG_MOVE_ONLY | ctm.CTM_FLAG_PROFILE, stream=stream, device=dev)
        A = torch.from_numpy(g["A"]).to(dev)
        B = torch.from_numpy(g["B"]).to(dev)
        env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi, device=dev)
        flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
        iso = torch.zeros(h.iso_numel(), dtype=torch.float64, device=dev)
    F_move = ctm.ctm_move_flops(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp)

    def ev():
        return torch.cuda.Event(enable_timing=True)

    def step(inject=False, handle=h, stats=None, env=env):
        flush.zero_()
        e0, e1 = ev(), ev()
        e0.record(stream)
        st = handle.ctm_left_move(A, B, env, iso_in=iso if inject else None, iso_out=None if inject else iso)
        e1.record(stream)
        e1.synchronize()
        if stats is not None:
            stats.append(st)
        return e0.elapsed_time(e1)

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            step()
        k0 = h.kernel_count
        stats = []
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        with ClockSampler(local) as clk:
            ms = []
            for i in range(args.steps):
                # CTM_BENCH_PROFILE=1: ncu --profile-from-start off captures the first timed step
                # (the launch list under profiles/ comes from this command)
                prof = i == 0 and os.environ.get("CTM_BENCH_PROFILE") == "1"
                if prof:
                    torch.cuda.profiler.start()
                ms.append(step(stats=stats))
                if prof:
                    torch.cuda.profiler.stop()
        torch.cuda.synchronize()
        launches = h.kernel_count - k0
        # CTM_FLAG_WARM_START (off in the headline above): the SAME sequence of moves -- a fresh copy of
        # the initial environment, the same warm-up and timed steps -- on a handle whose truncating
        # solves start from their site's previous block.  Every solve is still certified on its own
        # matrix (tests: shadowed trajectories with the flag on); reported beside the cold number.
        wstats, ms_w, warm_err = [], [], None
        try:
            hw = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp, svd_algo=svd,
                               flags=ctm.CTM_FLAG_MOVE_ONLY | ctm.CTM_FLAG_WARM_START, stream=stream, device=dev)
            env_w = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi, device=dev)
            for _ in range(max(args.warmup, 3)):
                step(handle=hw, env=env_w)
            ms_w = [step(handle=hw, env=env_w, stats=wstats) for _ in range(args.steps)]
            torch.cuda.synchronize()
            del hw, env_w
        except Exception as e:   # an opt-in extra must not cost the bench line
            warm_err = repr(e)
        # contraction-only (isometries injected: no reduced env, no SVD) -- the hot contraction
        for _ in range(2):
            step(inject=True)
        ms_c = [step(inject=True) for _ in range(args.steps)]
        # the same contraction-only move replayed from a CUDA graph (SURVEY 8(d) protocol 3)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            h.ctm_left_move(A, B, env, iso_in=iso, stats=False)
        graph.replay()
        stream.synchronize()
        ms_g = []
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = ev(), ev()
            e0.record(stream)
            graph.replay()
            e1.record(stream)
            e1.synchronize()
            ms_g.append(e0.elapsed_time(e1))
        del graph
        # per-launch profile of tc_gemm: the contraction-only step, and the full step (the
        # isometry solvers' GEMMs on the worker streams included)
        pst = []
        for _ in range(3):
            step(inject=True, handle=hp, stats=pst)
        pfull = []
        for _ in range(3):
            step(inject=False, handle=hp, stats=pfull)
        # rows a1, a3, a4 timed alone: the reduced environment of each cut type with its side
        # isometries injected (no SVD) -- half of the method's flops, otherwise only measured
        # inside the isometry stage on the worker streams
        renv = {}
        for x, X in (("a", A), ("b", B)):
            M = torch.empty(cfg.chi * cfg.D * cfg.D * cfg.chi, dtype=torch.float64, device=dev)
            n1 = min(cfg.chi_pp, cfg.chi * cfg.D)
            n2 = min(cfg.chi_pp, n1 * cfg.D)
            side = torch.empty(2 * (cfg.chi * cfg.D * n1 + n1 * cfg.D * n2), dtype=torch.float64, device=dev)
            rargs = (env.C[(x, 1)], env.T[(x, 2)], env.C[(x, 2)], env.T[(x, 1)], X, X, env.T[(x, 3)], M)
            h.ctm_reduced_env(*rargs, iso_out=side)
            renv[x] = (rargs, side)
        ms_r = []
        for i in range(2 + 2 * args.steps):
            x = "ab"[i % 2]
            flush.zero_()
            e0, e1 = ev(), ev()
            e0.record(stream)
            h.ctm_reduced_env(*renv[x][0], iso_in=renv[x][1])
            e1.record(stream)
            e1.synchronize()
            if i >= 2:
                ms_r.append(e0.elapsed_time(e1))
        # end to end through the C ABI with HOST buffers (pinned), copies inside the timed region:
        # every step uploads its inputs (A, B, the 16 environment tensors) and reads back the 16
        # updated tensors.  Steps are independent problems, so the copies are double-buffered on
        # a copy stream: step i+1's upload and step i's read-back overlap step i+1 / i's move.
        pinned = {"A": torch.from_numpy(g["A"]).pin_memory(), "B": torch.from_numpy(g["B"]).pin_memory()}
        hC = {k: torch.from_numpy(v.reshape(-1)).pin_memory() for k, v in g["C"].items()}
        hT = {k: torch.from_numpy(v.reshape(-1)).pin_memory() for k, v in g["T"].items()}
        oC = [{k: torch.empty_like(v).pin_memory() for k, v in hC.items()} for _ in range(2)]
        oT = [{k: torch.empty_like(v).pin_memory() for k, v in hT.items()} for _ in range(2)]
        h2d = sum(t.numel() * 8 for t in list(pinned.values()) + list(hC.values()) + list(hT.values()))
        d2h = sum(t.numel() * 8 for t in list(oC[0].values()) + list(oT[0].values()))
        sets = [{"A": torch.empty_like(A), "B": torch.empty_like(B),
                 "env": ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi, device=dev)} for _ in range(2)]
        cstream = torch.cuda.Stream(dev)

        def e2e_run(n):
            up = [ev() for _ in range(2)]
            moved = [ev() for _ in range(2)]
            down = [ev() for _ in range(2)]
            t_begin, t_end = ev(), ev()

            def upload(j):
                st_ = sets[j]
                with torch.cuda.stream(cstream):
                    st_["A"].copy_(pinned["A"], non_blocking=True)
                    st_["B"].copy_(pinned["B"], non_blocking=True)
                    for k in hC:
                        st_["env"].C[k][: hC[k].numel()].copy_(hC[k], non_blocking=True)
                        st_["env"].T[k][: hT[k].numel()].copy_(hT[k], non_blocking=True)
                    up[j].record(cstream)

            t_begin.record(cstream)
            upload(0)
            for i in range(n):
                j = i % 2
                stream.wait_event(up[j])
                if i + 1 < n:   # next step's upload: its buffers were last read back at step i - 1
                    if i >= 1:
                        cstream.wait_event(down[1 - j])
                    upload(1 - j)
                flush.zero_()
                h.ctm_left_move(sets[j]["A"], sets[j]["B"], sets[j]["env"])
                moved[j].record(stream)
                cstream.wait_event(moved[j])
                with torch.cuda.stream(cstream):
                    for k in hC:
                        oC[j][k].copy_(sets[j]["env"].C[k][: oC[j][k].numel()], non_blocking=True)
                        oT[j][k].copy_(sets[j]["env"].T[k][: oT[j][k].numel()], non_blocking=True)
                    down[j].record(cstream)
            t_end.record(cstream)
            t_end.synchronize()
            return t_begin.elapsed_time(t_end) / n

        e2e_run(2)
        ms_e2e = [e2e_run(max(3, args.steps // 2))]

    t_step = float(np.mean(ms))
    t_c = float(np.mean(ms_c))
    t_e2e = float(np.mean(ms_e2e))
    t_g = float(np.mean(ms_g))
    t_step, t_c, t_e2e, t_g = max_over_ranks([t_step, t_c, t_e2e, t_g], device=dev)
    ms_svd = float(np.mean([s["ms_svd"] for s in stats]))
    ms_iso = float(np.mean([s["ms_isometry"] for s in stats]))
    gem_ms = float(np.mean([s["ms_gemm"] for s in pst]))
    gem_fl = float(np.mean([s["gemm_flops"] for s in pst]))
    gem_n = float(np.mean([s["gemm_launches"] for s in pst]))
    achieved = gem_fl / (gem_ms * 1e-3) / 1e12
    full_ms = float(np.mean([s["ms_gemm"] for s in pfull]))
    full_fl = float(np.mean([s["gemm_flops"] for s in pfull]))
    full_n = float(np.mean([s["gemm_launches"] for s in pfull]))
    full_achieved = full_fl / (full_ms * 1e-3) / 1e12
    jac_ms = float(np.mean([s["ms_jacobi"] for s in stats]))
    jac_n = float(np.mean([s["n_jacobi"] for s in stats]))
    t_renv = float(np.mean(ms_r))
    F_renv = renv_flops(cfg)
    k7_ms = float(np.mean([s["ms_commit"] for s in pst]))
    k7_bytes = float(np.mean([s["commit_bytes"] for s in pst]))
    k7_n = float(np.mean([s["n_commit"] for s in pst]))
    hbm = hbm_peak_gbs()
    if rank != 0:
        return
    value = job_value(world, t_step)
    line = {
        "metric": METRIC, "value": value, "unit": "moves/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": t_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, ctm_inputs.py)",
        "config": {"workload": workload(cfg), "D": cfg.D, "chi": cfg.chi, "svd": args.svd,
                   "parallelism": f"replicas{world}",
                   "l2": "256 MB L2 flush between timed steps; intermediates > L2"},
        "ms_isometry_stage_per_move": ms_iso, "ms_svd_calls_summed_per_move": ms_svd,
        "svd_fallbacks_per_move": float(np.mean([s.get("n_svd_fallback", 0) for s in stats])),
        "ms_absorb_per_move": t_step - ms_iso,
        "contraction_only": {"moves_per_s": job_value(world, t_c), "ms_per_move": t_c,
                             "flops_per_move": gem_fl, "tflops": gem_fl / (t_c * 1e-3) / 1e12,
                             "frac_of_fp64_peak": gem_fl / (t_c * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                             "note": "isometries injected (INJECT_ISO): chains + corners + commit only, "
                                     "no reduced env, no SVD"},
        "contraction_only_graph": {"moves_per_s": job_value(world, t_g), "ms_per_move": t_g,
                                   "tflops": gem_fl / (t_g * 1e-3) / 1e12,
                                   "frac_of_fp64_peak": gem_fl / (t_g * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                                   "note": "the same move captured once in a CUDA graph and replayed"},

        "flops_per_move": F_move,
        "tflops_full_move": F_move / (t_step * 1e-3) / 1e12,
        # headline roofline: the method's algorithmic flops per step (SURVEY 8(a) closed form F_move, rows
        # a1-a11; the isometry solver's own GEMMs are NOT counted) over the device time of the whole step
        "roofline": {"bound": "tensor", "kernel": "whole left move (rows a1-a11: reduced envs, isometry solves, "
                                                  "chains, corners, commit)",
                     "achieved": F_move / (t_step * 1e-3) / 1e12, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": F_move / (t_step * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, "traffic": None,
                     "flops_per_step": F_move, "ms_per_step": t_step,
                     "peak_source": "measured DMMA loop (profiles/r01_probe_fp64.txt); MEASURED_PEAKS.json has no FP64"},
        # rows a1, a3, a4 alone (side isometries injected): the other half of the method's flops
        "roofline_renv": {"bound": "tensor", "kernel": "tc_gemm, one reduced environment (rows a1, a3, a4 + v1^T Q), "
                                                       "side isometries injected",
                          "achieved": F_renv / (t_renv * 1e-3) / 1e12, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                          "frac": F_renv / (t_renv * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, "traffic": None,
                          "flops_per_call": F_renv, "ms_per_call": t_renv, "calls_per_move": 4,
                          "note": "CUDA events around ctm_reduced_env(iso_in) on the library stream, L2 flushed"},
        # K7: Frobenius normalise + commit of the six new tensors, HBM-bound
        "roofline_commit": ({"bound": "hbm", "kernel": "scale_commit_kernel (K7)",
                             "achieved": k7_bytes / (k7_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                             "frac": (k7_bytes / (k7_ms * 1e-3) / 1e9 / hbm) if hbm else None, "traffic": None,
                             "bytes_per_step": k7_bytes, "ms_per_step": k7_ms, "launches_per_step": k7_n,
                             "peak_source": "MEASURED_PEAKS.json hbm_gbs"} if k7_ms > 0 else None),
        # the isometry solver (rows a2, a5 SVDs) is reported in ms, not as a flop rate
        "solver": {"ms_isometry_stage_per_move": ms_iso, "ms_svd_calls_summed_per_move": ms_svd,
                   "ms_jacobi_summed_per_move": jac_ms, "jacobi_launches_per_move": jac_n,
                   "solver_and_contraction_gemm_ms_summed": full_ms, "gemm_flops_summed": full_fl,
                   "gemm_launches": full_n,
                   "note": "isometry stage = wall time of rows a1-a5 (fork to join); solver GEMM flops are not the "
                           "method's flops"},
        "truncation_gaps": {"main_cut_gap[absorption][ab,ba]": stats[0]["cut_gap"],
                            "side_gap[absorption][a-l,a-r,b-l,b-r]": stats[0]["side_gap"],
                            "min_gap": float(np.min([s["min_gap"] for s in stats]))},
        "roofline_contraction": {"bound": "tensor", "kernel": "tc_gemm (FP64 DMMA.8x8x4)", "achieved": achieved,
                     "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                     "traffic": traffic_bytes(cfg), "traffic_unit": "DRAM bytes per step (ncu, profiles/r02_traffic.json)",
                     "launches_per_step": gem_n, "ms_per_step": gem_ms,
                     "peak_source": "measured DMMA loop (profiles/r01_probe_fp64.txt); MEASURED_PEAKS.json has no FP64"},
        "e2e": {"value": job_value(world, t_e2e), "unit": "moves/s", "h2d_bytes_per_step": h2d,
                "pipelining": "inputs uploaded and results read back on a copy stream, double-buffered across "
                              "independent steps (each step a move from host inputs)",
                "d2h_bytes_per_step": d2h},
        "warm_start": ({"error": warm_err} if warm_err or not ms_w else {
            "flag": "CTM_FLAG_WARM_START (opt-in; the headline value above is measured WITHOUT it)",
            "ms_per_step": float(np.mean(ms_w)), "moves_per_s": job_value(world, float(np.mean(ms_w))),
            "ms_steps": [round(x, 2) for x in ms_w], "cold_ms_steps": [round(x, 2) for x in ms],
            "warm_solves_per_move": float(np.mean([s["n_warm"] for s in wstats])),
            "certified_at_first_check_per_move": float(np.mean([s["n_warm_hit"] for s in wstats])),
            "cold_retries": int(np.sum([s["n_warm_retry"] for s in wstats])),
            "svd_fallbacks": int(np.sum([s["n_svd_fallback"] for s in wstats])),
            "note": "same move sequence as the headline (fresh copy of the initial environment, same warm-up, same "
                    "timed steps, L2 flushed); each truncating solve may start from its site's previous final block "
                    "and ends on the residual certificate of the new matrix.  On these synthetic (non-converging) "
                    "environments only the right-side cuts -- whose matrices repeat in consecutive LEFT moves -- "
                    "are certified at once; the other sites' first checks are wasted and they back off "
                    "(DESIGN.md 6).  Rank 0's own time (not max over ranks)"}),
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline:
        s = run_oracle_sample(cfg)
        line["cpu_baseline"] = {"value": 1.0 / s, "unit": "moves/s", "cores": host_cores(), "kind": "oracle",
                                "sample": f"1 full left move of {cfg.name} (NumPy/OpenBLAS fp64 oracle, {s:.1f} s)"}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    cfg = ci.CONFIGS[args.config]
    if args.impl == "reference":
        bench_reference(args, cfg)
    else:
        bench_ours(args, cfg)


if __name__ == "__main__":
    main()

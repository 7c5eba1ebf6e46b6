"""The TMA-staged contraction kernel (csrc/tc_gemm_tma.cuh) against the cp.async kernel.

Both kernels issue the same DMMA sequence on the same fragments (only the way a k-tile reaches
shared memory differs, and edges / the K tail arrive as TMA zero-fill instead of explicit zero
stores), so a whole left move with injected isometries must come out bit-identical with
CTM_TC_TMA=0 and with the default (TMA for the eligible chain steps S1, S3, S4, S6 and the corner
GEMMs at C4).  Each arm runs in its own process (the switch is read once per process).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import ctm_inputs as ci
from paper_2306_08212_b200 import ctm
cfg = ci.CONFIGS[sys.argv[2]]
g = ci.generate(cfg)
h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp, flags=ctm.CTM_FLAG_MOVE_ONLY)
# isometries: seeded random orthonormal columns (the contractions do not need SVD isometries)
rng = np.random.default_rng(7)
parts = []
for _ in range(4):
    q1, _ = np.linalg.qr(rng.standard_normal((cfg.chi * cfg.D, cfg.chi_p)))
    q2, _ = np.linalg.qr(rng.standard_normal((cfg.chi_p * cfg.D, cfg.chi)))
    parts += [q1.ravel(), q2.ravel()]
iso = torch.from_numpy(np.concatenate(parts)).cuda()
A = torch.from_numpy(g["A"]).cuda()
B = torch.from_numpy(g["B"]).cuda()
env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
h.ctm_left_move(A, B, env, iso_in=iso)
out = env.to_host()
np.savez(sys.argv[3], **{f"{k}_{key[0]}{key[1]}": v for k in ("C", "T") for key, v in out[k].items()})
"""


def _run(tmp_path, name, config, tma):
    env = dict(os.environ)
    env.pop("CTM_TC_TMA", None)
    if not tma:
        env["CTM_TC_TMA"] = "0"
    path = str(tmp_path / f"{name}.npz")
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, config, path], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(path)


@pytest.mark.parametrize("config", ["c4", "c5"])
def test_tma_kernel_is_bit_identical_to_the_cp_async_kernel(tmp_path, config):
    a = _run(tmp_path, "tma", config, True)
    b = _run(tmp_path, "cpasync", config, False)
    assert sorted(a.files) == sorted(b.files) and len(a.files) == 16
    for k in a.files:
        assert np.isfinite(a[k]).all()
        assert np.array_equal(a[k], b[k]), k

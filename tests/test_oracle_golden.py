"""Regression fixture of the oracle: tests/golden/oracle_small.json was written by
tools/make_golden.py from oracle/ only (never the CUDA path).  Re-running the oracle on the
same seeded inputs must reproduce it, so an accidental change of the oracle's arithmetic
fails here (a deliberate one regenerates the file and names its reason in the commit).

Tolerances follow the problem's conditioning: one left move / one iteration
of Tiny and one left move of C2 are reproducible to rounding; the C2 20-iteration values
amplify BLAS summation-order differences by ~1e13 and are recorded for information only."""
import json
import os

import numpy as np
import pytest

import ctm_inputs as ci
from oracle import ctm_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_small.json")


def _obs(env, A, B):
    h = ci.heisenberg_h()
    return {"norm_2x2": O.norm_2x2(env, A, B), "e_H": O.bond_energy(env, A, B, h, "H")[0],
            "e_V": O.bond_energy(env, A, B, h, "V")[0]}


@pytest.mark.parametrize("name,rtol", [("tiny", 1e-9), ("c2", 1e-6)])
def test_oracle_reproduces_golden_left_move(name, rtol):
    gold = json.load(open(GOLD))[name]
    cfg = ci.CONFIGS[name]
    g = ci.generate(cfg)
    assert (gold["seed"], gold["D"], gold["chi"]) == (cfg.seed, cfg.D, cfg.chi)
    e1 = O.left_move({"C": g["C"], "T": g["T"]}, g["A"], g["B"], cfg.chi, cfg.chi_p, cfg.chi_pp)
    got = _obs(e1, g["A"], g["B"])
    for k, v in gold["after_left_move"].items():
        assert got[k] == pytest.approx(v, rel=rtol, abs=1e-14), k


def test_oracle_reproduces_golden_tiny_iteration():
    gold = json.load(open(GOLD))["tiny"]
    cfg = ci.CONFIGS["tiny"]
    g = ci.generate(cfg)
    e = O.ctm_iteration({"C": g["C"], "T": g["T"]}, g["A"], g["B"], cfg.chi, cfg.chi_p, cfg.chi_pp)
    got = _obs(e, g["A"], g["B"])
    for k, v in gold["after_1_iterations"].items():
        assert np.isclose(got[k], v, rtol=1e-9, atol=1e-14), k

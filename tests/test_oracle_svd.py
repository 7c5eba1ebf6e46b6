"""Pins of the oracle's truncated SVD and two-stage isometry (SURVEY 8(c) 'TS / isometries').

These run on CPU (-m "not gpu")."""
import json
import os

import numpy as np
import pytest

from oracle import ctm_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_rank1_analytic():
    g = _gold("svd_cases.json")["rank1"]
    u, v = np.array(g["u"]), np.array(g["v"])
    m = np.outer(u, v)
    stats = []
    U = O.left_singular(m, 1, stats)
    assert np.isclose(stats[0]["sigma_first"], g["sigma"], rtol=1e-14)
    # the kept vector is u/|u| with the sign rule (largest entry positive)
    assert np.allclose(U[:, 0], u / np.linalg.norm(u), atol=1e-14)


def test_diag321_truncation():
    g = _gold("svd_cases.json")["diag321"]
    m = np.array(g["matrix"])
    stats = []
    U = O.left_singular(m, g["keep"], stats)
    assert np.allclose(U, np.array(g["left_vectors_after_sign_rule"]), atol=1e-15)
    kept = U.T @ m
    assert np.allclose(np.linalg.svd(kept, compute_uv=False), g["kept_sigma"])
    discarded = np.linalg.norm(m) ** 2 - np.linalg.norm(kept) ** 2
    assert np.isclose(discarded, g["discarded_weight"], atol=1e-14)


def test_sign_rule():
    rng = np.random.default_rng(3)
    U, _ = np.linalg.qr(rng.standard_normal((9, 4)))
    F = O.sign_fix(-U)
    for j in range(4):
        i = np.argmax(np.abs(F[:, j]))
        assert F[i, j] > 0
    assert np.allclose(np.abs(F), np.abs(U))
    # ties: lowest index wins
    T = np.array([[-1.0], [1.0]]) / np.sqrt(2)
    assert O.sign_fix(T)[0, 0] > 0


@pytest.mark.parametrize("shape,c1,c2", [((4, 2, 2, 4), 5, 3), ((3, 3, 3, 5), 4, 4), ((2, 2, 2, 2), 8, 8)])
def test_ts_isometry_properties(shape, c1, c2):
    rng = np.random.default_rng(11)
    Q = rng.standard_normal(shape)
    v1, v2 = O.ts_isometry(Q, c1, c2)
    P, K, B, F = shape
    n1 = min(c1, P * K)
    n2 = min(c2, n1 * B)
    assert v1.shape == (P, K, n1) and v2.shape == (n1, B, n2)
    m1 = v1.reshape(P * K, n1)
    m2 = v2.reshape(n1 * B, n2)
    assert np.allclose(m1.T @ m1, np.eye(n1), atol=1e-12)
    assert np.allclose(m2.T @ m2, np.eye(n2), atol=1e-12)
    V = O.compose_isometry(v1, v2).reshape(P * K * B, n2)
    assert np.allclose(V.T @ V, np.eye(n2), atol=1e-12)
    Pm = V @ V.T
    assert np.allclose(Pm @ Pm, Pm, atol=1e-12)


def test_ts_first_stage_is_best_rank_c1():
    """v1 spans the top-c1 left singular space of Q as (p,k) x (b,q) (Eckart-Young):
    the captured weight equals the sum of the c1 largest sigma^2."""
    rng = np.random.default_rng(5)
    Q = rng.standard_normal((5, 3, 3, 4))
    v1, _ = O.ts_isometry(Q, 6, 4)
    m = Q.reshape(15, 12)
    s = np.linalg.svd(m, compute_uv=False)
    cap = np.linalg.norm(v1.reshape(15, 6).T @ m) ** 2
    assert np.isclose(cap, np.sum(s[:6] ** 2), rtol=1e-12)


def test_sequential_full_chi_prime_equals_reduced():
    """SEQUENTIAL(chi' = chi D) == REDUCED given the same exact M (SURVEY 8(c) pin):
    with v1 square orthogonal, TS's composite V spans the top-chi left singular space of
    M grouped (p,k,b) x q, so the projectors agree."""
    rng = np.random.default_rng(7)
    chi, D = 4, 2
    M = rng.standard_normal((chi, D, D, chi))
    for keep in (1, 2, 3):
        v1, v2 = O.ts_isometry(M, chi * D, keep)
        V = O.compose_isometry(v1, v2).reshape(chi * D * D, keep)
        Vr = O.one_shot_isometry(M, keep).reshape(chi * D * D, keep)
        assert np.allclose(V @ V.T, Vr @ Vr.T, atol=1e-12)


def test_full_rows_gives_identity_projector():
    """Reading R11: n == rows keeps the full U (square orthogonal) -> P = I even when
    rank < rows (no-truncation case)."""
    rng = np.random.default_rng(9)
    Q = rng.standard_normal((2, 2, 2, 1))        # Q2 stage is 4 x 1: rank 1, rows 4
    v1, v2 = O.ts_isometry(Q, 4, 8)
    V = O.compose_isometry(v1, v2).reshape(8, -1)
    assert V.shape == (8, 8)
    assert np.allclose(V @ V.T, np.eye(8), atol=1e-12)

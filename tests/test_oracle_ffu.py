"""Pins of the imaginary-time / fast-full-update oracle (oracle/ffu_oracle.py; SURVEY 8(f)
item 4).  Each function is checked against something other than itself: closed
forms (the singlet/triplet gate, product eigenstates), exact identities (reductions,
untruncated splits), an independent contraction (bond environment vs the bond-rho closure
of ctm_oracle), and the variational property of ALS."""
import numpy as np
import pytest

import ctm_inputs as ci
from oracle import ctm_oracle as O
from oracle import ffu_oracle as F


def _rand_case(seed, d=2, D=2, chi=4):
    cfg = ci.custom(d, D, chi, seed_index=seed)
    g = ci.generate(cfg)
    return {"C": g["C"], "T": g["T"]}, g["A"], g["B"]


# ---- R25 gate ---------------------------------------------------------------------------
def test_gate_heisenberg_singlet_triplet_closed_form():
    """h = S.S has the singlet at -3/4 and the triplet at +1/4: exp(-delta h) =
    e^{-delta/4} (1 - P_s) + e^{3 delta/4} P_s, P_s = |s><s|, |s> = (|01> - |10>)/sqrt 2."""
    h = ci.heisenberg_h()
    delta = 0.3
    s = np.array([0.0, 1.0, -1.0, 0.0]) / np.sqrt(2.0)
    Ps = np.outer(s, s)
    want = np.exp(-delta / 4) * (np.eye(4) - Ps) + np.exp(3 * delta / 4) * Ps
    assert np.allclose(F.trotter_gate(h, delta).reshape(4, 4), want, atol=1e-14)


def test_gate_identity_limit_and_inverse():
    h = ci.heisenberg_h()
    assert np.allclose(F.trotter_gate(h, 0.0).reshape(4, 4), np.eye(4), atol=1e-15)
    g, gi = F.trotter_gate(h, 0.1).reshape(4, 4), F.trotter_gate(h, -0.1).reshape(4, 4)
    assert np.allclose(g @ gi, np.eye(4), atol=1e-14)


# ---- R26 reductions ---------------------------------------------------------------------
@pytest.mark.parametrize("D", [2, 3])
def test_reductions_are_exact_and_isometric(D):
    _, A, B = _rand_case(61, D=D)
    X, aR = F.reduce_left(A)
    bL, Y = F.reduce_right(B)
    assert np.allclose(np.einsum("uldw,wsr->suldr", X, aR), A, atol=1e-14)
    assert np.allclose(np.einsum("slv,vudr->suldr", bL, Y), B, atol=1e-14)
    Xm = X.reshape(-1, X.shape[-1])
    Ym = Y.reshape(Y.shape[0], -1)
    assert np.allclose(Xm.T @ Xm, np.eye(Xm.shape[1]), atol=1e-13)
    assert np.allclose(Ym @ Ym.T, np.eye(Ym.shape[0]), atol=1e-13)


# ---- R27 bond environment ---------------------------------------------------------------
def test_bond_env_closes_to_the_bond_rho_trace():
    """sum N(w,v,w',v') theta(w,s,t,v) theta(w',s,t,v') with theta = aR bL (the unreduced
    bond) equals the trace of ctm_oracle.bond_rho on the same window -- an independent
    contraction of the same network."""
    env, A, B = _rand_case(62, D=2, chi=5)
    X, aR = F.reduce_left(A)
    bL, Y = F.reduce_right(B)
    N = F.bond_env_h(env, X, Y)
    th = np.einsum("wsr,trv->wstv", aR, bL)
    got = np.einsum("wstv,wvxy,xsty->", th, N, th)
    rho = O.bond_rho(env, A, B, "H")
    want = np.einsum("stst->", rho)
    assert got == pytest.approx(want, rel=1e-11)


def test_positivise_keeps_a_positive_N_and_clips_a_negative_one():
    rng = np.random.default_rng(3)
    Z = rng.standard_normal((6, 6))
    P = (Z @ Z.T).reshape(2, 3, 2, 3)
    assert np.allclose(F.positivise(P), P, atol=1e-10)
    M = F.positivise((-(Z @ Z.T)).reshape(2, 3, 2, 3)).reshape(6, 6)
    assert np.linalg.eigvalsh(M).min() >= 0.0


# ---- R28 split --------------------------------------------------------------------------
def test_untruncated_bond_update_applies_the_gate_exactly():
    """With the new bond as large as the gated pair's rank, the truncated-SVD split (R28's
    start) is exact: the updated pair contracted over its bond is the gate applied to the old
    pair (up to normalisation).  ALS from there keeps the N-weighted error at zero (it may move
    the pair along N's near-null directions, which the metric does not see)."""
    env, A, B = _rand_case(63, D=2, chi=4)
    g = F.trotter_gate(ci.heisenberg_h(), 0.2)
    A2, B2, _ = F.bond_update_h(env, A, B, g, D=8, sweeps=0)        # rank <= (d m) = 8: keep all
    old = np.einsum("suldr,tRrDe->stuldRDe", A, B)                  # (sA, sB, A's u,l,d, B's u,d,r)
    want = np.einsum("stpq,pqabcxyz->stabcxyz", g, old)
    got = np.einsum("suldr,tRrDe->stuldRDe", A2, B2)
    want, got = want / np.linalg.norm(want), got / np.linalg.norm(got)
    assert min(np.abs(got - want).max(), np.abs(got + want).max()) <= 1e-12
    X, aR = F.reduce_left(A)
    bL, Y = F.reduce_right(B)
    N = F.positivise(F.bond_env_h(env, X, Y))
    th = F.apply_gate(aR, bL, g)
    _, _, costs = F.als_split(th, N, 8, sweeps=3)
    assert max(abs(c) for c in costs) <= 1e-12 * np.einsum("wstv,wvxy,xsty->", th, N, th)


def test_als_never_increases_the_environment_weighted_error():
    """ALS (R28) minimises exactly over one factor per half-step: the N-weighted error is
    non-increasing and never worse than the truncated-SVD start."""
    env, A, B = _rand_case(64, D=3, chi=6)
    X, aR = F.reduce_left(A)
    bL, Y = F.reduce_right(B)
    N = F.positivise(F.bond_env_h(env, X, Y))
    th = F.apply_gate(aR, bL, F.trotter_gate(ci.heisenberg_h(), 0.4))
    a0, b0 = F.svd_split(th, 2)
    phi = np.einsum("wsr,trv->wstv", a0, b0)
    e0 = np.einsum("wstv,wvxy,xsty->", phi - th, N, phi - th)
    _, _, costs = F.als_split(th, N, 2, sweeps=6)
    assert costs[0] <= e0 * (1 + 1e-10)
    for c0, c1 in zip(costs, costs[1:]):
        assert c1 <= c0 * (1 + 1e-9) + 1e-15


def test_product_eigenstate_is_invariant():
    """D = 1, zz gate (diagonal), z-polarised product state: an eigenstate of every gate, so
    the update returns the same state (SPEC S:L386-style closed form)."""
    d, D = 2, 1
    up = np.zeros((d, 1, 1, 1, 1))
    up[0] = 1.0
    sz = np.diag([1.0, -1.0])
    hzz = np.einsum("ac,bd->abcd", sz, sz)
    env, _, _ = _rand_case(65, D=1, chi=2)
    for bond in ("H1", "H2", "V1", "V2"):
        A2, B2, _ = F.bond_update(env, up, up, F.trotter_gate(hzz, 0.3), 1, 3, bond)
        assert np.allclose(np.abs(A2), up, atol=1e-14) and np.allclose(np.abs(B2), up, atol=1e-14)


@pytest.mark.parametrize("bond", ["H1", "H2", "V1", "V2"])
def test_zero_time_step_leaves_every_bond_unchanged(bond):
    """delta = 0: the gate is the identity and the pair already has bond D, so each update
    returns the same two-site state (up to the new bond's gauge and normalisation)."""
    env, A, B = _rand_case(66, D=2, chi=4)
    A2, B2, _ = F.bond_update(env, A, B, F.trotter_gate(ci.heisenberg_h(), 0.0), 2, 4, bond)
    pair = {"H1": "suldr,tRrDe->stuldRDe", "H2": "surde,tRLDr->stRLDude",
            "V1": "suldr,tdLDR->stulrLDR", "V2": "sdlDr,tULdR->stULRlDr"}[bond]
    old = np.einsum(pair, A, B)
    new = np.einsum(pair, A2, B2)
    old, new = old / np.linalg.norm(old), new / np.linalg.norm(new)
    assert min(np.abs(new - old).max(), np.abs(new + old).max()) <= 1e-10


# ---- R29/R30 Trotter step -----------------------------------------------------------------
def test_heisenberg_evolution_goes_below_every_product_state():
    """Imaginary-time evolution of the AFM Heisenberg model at D = 2: the
    energy per site falls below -1/2, the minimum over product states (Neel: -1/4 per bond,
    two bonds per site), towards the D = 2 variational value (~ -0.65)."""
    D, chi = 2, 8
    cfg = ci.custom(2, D, chi, seed_index=67)
    g = ci.generate(cfg, "double_layer")
    A, B = g["A"], g["B"]
    env = {"C": g["C"], "T": g["T"]}
    for _ in range(5):
        env = O.ctm_iteration(env, A, B, chi)
    h = ci.heisenberg_h()
    es = []
    for step in range(60):
        env, A, B, _ = F.trotter_step(env, A, B, h, 0.1 if step < 40 else 0.05, D, chi, sweeps=3)
        eH = O.bond_energy(env, A, B, h, "H")[0]
        eV = O.bond_energy(env, A, B, h, "V")[0]
        es.append(eH + eV)
    print("energy per site", es[0], es[9], es[-1])
    assert es[-1] < -0.5
    assert es[-1] < es[0]

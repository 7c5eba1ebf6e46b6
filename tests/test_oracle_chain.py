"""Pins of the oracle's absorb/truncate chain, corner growth and reduced environment
(SURVEY 8(c) rows 'Chains and corners (a6-a9)' and 'Approx reduced env (a1-a4)').

Brute force here = ONE np.einsum over the whole network with optimize=False (plain
nested loops, no pairwise order), at tiny sizes."""
import numpy as np
import pytest

import ctm_inputs as ci
from oracle import ctm_oracle as O


def _rand(rng, *shape):
    return rng.standard_normal(shape)


def _isos(rng, chi, D, chi_p, chi_out):
    return ci.random_isometries(rng, chi, D, chi_p, chi_out)


def test_chain_matches_whole_network_einsum():
    rng = np.random.default_rng(1)
    chi, D, d, cp = 3, 2, 2, 3
    T = _rand(rng, chi, D, D, chi)
    X = _rand(rng, d, D, D, D, D)
    Xb = _rand(rng, d, D, D, D, D)
    v1i, v2i = _isos(rng, chi, D, cp, chi)
    v1o, v2o = _isos(rng, chi, D, cp, chi)
    got = O.absorb_truncate(T, X, Xb, v1i, v2i, v1o, v2o)
    # T'(o1,kz,bz,o2) = v1_in(p,ki,a) v2_in(a,bi,o1) T(p,kf,bf,q) X(s,ki,kf,ko,kz)
    #                   X*(s,bi,bf,bo,bz) v1_out(q,ko,c) v2_out(c,bo,o2)
    want = np.einsum("pia,ajx,pfgq,sifoz,sjgbw,qoc,cby->xzwy",
                     v1i, v2i, T, X, Xb, v1o, v2o, optimize=False)
    assert np.allclose(got, want, rtol=0, atol=1e-13 * np.abs(want).max())


def test_chain_sequential_equals_one_shot_with_composed_isometry():
    """Contraction-order independence: the sequential chain with (v1, v2)
    equals the one-shot chain with V = v1 v2."""
    rng = np.random.default_rng(2)
    chi, D, d, cp = 5, 3, 2, 4
    T = _rand(rng, chi, D, D, chi)
    X = _rand(rng, d, D, D, D, D)
    v1i, v2i = _isos(rng, chi, D, cp, 6)
    v1o, v2o = _isos(rng, chi, D, cp, 4)
    got = O.absorb_truncate(T, X, X, v1i, v2i, v1o, v2o)
    want = O.absorb_one_shot(T, X, X, O.compose_isometry(v1i, v2i), O.compose_isometry(v1o, v2o))
    assert got.shape == (6, D, D, 4)
    assert np.allclose(got, want, atol=1e-13 * np.abs(want).max())


def test_chain_bilinear_and_quadratic():
    rng = np.random.default_rng(3)
    chi, D, d = 4, 2, 2
    T = _rand(rng, chi, D, D, chi)
    X, Y = _rand(rng, d, D, D, D, D), _rand(rng, d, D, D, D, D)
    iso = (*_isos(rng, chi, D, 4, 4), *_isos(rng, chi, D, 4, 4))
    f = lambda a, b: O.absorb_truncate(T, a, b, *iso)
    a = 1.7
    assert np.allclose(f(a * X, Y), a * f(X, Y), atol=1e-13)
    assert np.allclose(f(X, a * Y), a * f(X, Y), atol=1e-13)
    assert np.allclose(f(X + Y, Y), f(X, Y) + f(Y, Y), atol=1e-13)
    assert np.allclose(f(a * X, a * X), a * a * f(X, X), atol=1e-13)


def test_corners_match_whole_network_einsum():
    rng = np.random.default_rng(4)
    chi, D, cp = 4, 2, 3
    C = _rand(rng, chi, chi)
    T = _rand(rng, chi, D, D, chi)
    v1, v2 = _isos(rng, chi, D, cp, 5)
    # C^1 (d=x, r=p), T^2 (l=p, k, b, r), new C^1'(o, r)
    want = np.einsum("xp,xka,pkbr,abo->or", C, v1, T, v2, optimize=False)
    assert np.allclose(O.corner_top_left(C, T, v1, v2), want, atol=1e-13)
    # C^4 (r=p, u=x), T^4 (r=r', k, b, l=p), new C^4'(r', o)
    want4 = np.einsum("px,xka,rkbp,abo->ro", C, v1, T, v2, optimize=False)
    assert np.allclose(O.corner_bottom_left(C, T, v1, v2), want4, atol=1e-13)
    V = O.compose_isometry(v1, v2)
    assert np.allclose(O.corner_top_left_one_shot(C, T, V), want, atol=1e-13)
    assert np.allclose(O.corner_bottom_left_one_shot(C, T, V), want4, atol=1e-13)


def _renv_inputs(rng, chi, D, d, sym=False):
    C1, C2 = _rand(rng, chi, chi), _rand(rng, chi, chi)
    T1, T2, T3 = (_rand(rng, chi, D, D, chi) for _ in range(3))
    X = _rand(rng, d, D, D, D, D)
    return C1, T2, C2, T1, X, X, T3


def test_reduced_env_exact_matches_whole_network_einsum():
    rng = np.random.default_rng(5)
    C1, T2, C2, T1, X, Xb, T3 = _renv_inputs(rng, 4, 2, 2)
    got = O.reduced_env_exact(C1, T2, C2, T1, X, Xb, T3)
    # picture legs: C1(r=p, d=x) T2(l=p, ku, bu, r=z) C2(l=z, d=y) T1(u=x, kl, bl, d=q)
    #               X(s,ku,kl,kd,kr) X*(s,bu,bl,bd,br) T3(u=y, kr, br, d=Q)
    want = np.einsum("xp,pkbz,zy,qlmx,sklKr,sbmBw,yrwQ->qKBQ",
                     C1, T2, C2, T1, X, Xb, T3, optimize=False)
    assert np.allclose(got, want, atol=1e-12 * np.abs(want).max())


def test_reduced_env_approx_untruncated_equals_exact():
    """chi'' >= chi D^2: side isometries are square orthogonal, P_l = P_r = I, so the
    approximated M equals the exact M entrywise."""
    rng = np.random.default_rng(6)
    chi, D = 4, 2
    C1, T2, C2, T1, X, Xb, T3 = _renv_inputs(rng, chi, D, 2)
    M, (vl1, vl2, vr1, vr2) = O.reduced_env_approx(C1, T2, C2, T1, X, Xb, T3, chi * D * D)
    assert vl2.shape[-1] == chi * D * D
    assert np.allclose(M, O.reduced_env_exact(C1, T2, C2, T1, X, Xb, T3), atol=1e-12)


def test_reduced_env_approx_exact_when_side_networks_have_low_rank():
    """Truncated but lossless side isometries: if T^1 and T^3 factor through a rank-r far
    leg, Q_l = C^1 T^1 has (p,k,b) x q rank <= r and (p,k) x (b,q) rank <= r*D, so
    TS(Q_l; c1 = r*D, c2 = r) keeps its whole range and M_approx == M_exact.  Detects
    isometries applied to the wrong legs (e.g. ket/bra swapped, T is NOT k<->b symmetric)."""
    rng = np.random.default_rng(8)
    chi, D, d, r = 4, 2, 2, 2
    C1, T2, C2, _, X, _, _ = _renv_inputs(rng, chi, D, d)
    Xb = _rand(rng, d, D, D, D, D)        # ket != bra: a ket/bra mix-up changes M
    def lowrank_T():                       # T(u,k,b,d) stored (d,k,b,u) = sum_i f_i(d) g_i(k,b,u)
        f = _rand(rng, chi, r)
        g = _rand(rng, r, D, D, chi)
        return np.einsum("qi,ikbu->qkbu", f, g)
    T1 = lowrank_T()
    T3s = lowrank_T()                      # (d,k,b,u) -> store as (u,k,b,d)
    T3 = T3s.transpose(3, 1, 2, 0)
    exact = O.reduced_env_exact(C1, T2, C2, T1, X, Xb, T3)
    M, (vl1, vl2, vr1, vr2) = O.reduced_env_approx(C1, T2, C2, T1, X, Xb, T3, r * D)
    # r*D = 4 < (p,k) rows 8; second stage keeps min(4, 4*D=8) = 4 > r: still lossless
    assert vl1.shape == (chi, D, r * D) and vl2.shape == (r * D, D, r * D)
    assert np.allclose(M, exact, atol=1e-12 * np.abs(exact).max())
    # and a genuinely lossy chi'' = 1 must NOT reproduce it
    M1, _ = O.reduced_env_approx(C1, T2, C2, T1, X, Xb, T3, 1)
    assert not np.allclose(M1, exact, atol=1e-3 * np.abs(exact).max())


def test_standard_half_network_closes_to_norm_2x2():
    """The STANDARD sub-network (upper half) contracted with the lower half (the same
    function on the 180-degree-rotated lattice) equals the 2x2 norm closure."""
    cfg = ci.custom(2, 2, 3, seed_index=41)
    g = ci.generate(cfg)
    env = {"C": g["C"], "T": g["T"]}
    A, B = g["A"], g["B"]
    C, T = env["C"], env["T"]
    up = O.half_network_standard(C[("a", 1)], T[("a", 2)], T[("b", 2)], C[("b", 2)], T[("a", 1)],
                                 A, A, B, B, T[("b", 3)])
    e2, A2, B2 = O.rotate_cw(*O.rotate_cw(env, A, B))
    C2, T2 = e2["C"], e2["T"]
    lo = O.half_network_standard(C2[("a", 1)], T2[("a", 2)], T2[("b", 2)], C2[("b", 2)],
                                 T2[("a", 1)], A2, A2, B2, B2, T2[("b", 3)])
    # up(q, kA, bA, kB, bB, q') ; lo(q'_, kA2, bA2, kB2, bB2, q_) with A2 under B, B2 under A
    val = np.einsum("qabcdQ,Qcdabq->", up, lo)
    assert np.isclose(val, O.norm_2x2(env, A, B), rtol=1e-11)

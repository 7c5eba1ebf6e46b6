"""Pins of the oracle's column absorption, left move and the rotated R/U/D moves
(SURVEY 8(c) 'Column absorption and move (a10, a11)').

No truncation (every TS keeps n = rows columns, so every V is square orthogonal and
P = V V^T = I): the new boundary column, contracted along its internal bonds, must equal
the old column contracted with the inserted column(s) of the lattice.  The inserted
columns are written out below directly in picture legs for each of the four directions,
independently of the oracle's rotate-by-relabelling, so these also pin the rotation."""
import numpy as np
import pytest

import ctm_inputs as ci
from oracle import ctm_oracle as O

E = lambda spec, *ops: np.einsum(spec, *ops, optimize="greedy")


# --- boundary columns/rows contracted along their internal bonds (storage orders) ---
def col_left(C1, Tt, Tb, C4):      # C1(d,r) T1(d,k,b,u) T1(d,k,b,u) C4(r,u) -> (R,k,b,m,n,S)
    return E("xR,yklx,zmny,Sz->RklmnS", C1, Tt, Tb, C4)


def col_right(C2, Tt, Tb, C3):     # C2(l,d) T3(u,k,b,d) T3 C3(u,l) -> (L,k,b,m,n,S)
    return E("Lx,xkly,ymnz,zS->LklmnS", C2, Tt, Tb, C3)


def row_up(C1, Tl, Tr, C2):        # C1(d,r) T2(l,k,b,r) T2 C2(l,d) -> (L,k,b,m,n,R)
    return E("Lx,xkly,ymnz,zR->LklmnR", C1, Tl, Tr, C2)


def row_down(C4, Tl, Tr, C3):      # C4(r,u) T4(r,k,b,l) T4 C3(u,l) -> (L,k,b,m,n,R)
    return E("xL,yklx,zmny,Rz->LklmnR", C4, Tl, Tr, C3)


# --- inserting one column/row of the lattice (site legs (s,u,l,d,r)) -------------------
def ins_left(col, T2, X, Y, T4):   # col (R,k,b,m,n,S); T2(l=R,..,r=R2); T4(r=S2,..,l=S)
    return E("RkbmnS,RuvQ,sukdK,svbeL,tdmgM,teniN,WgiS->QKLMNW",
             col, T2, X, X, Y, Y, T4)


def ins_right(col, T2, X, Y, T4):  # col (L,k,b,m,n,S); T2(l=Q, r=L); T4(r=S, l=W)
    return E("LkbmnS,QuvL,suKdk,svPeb,tdMgm,teNin,SgiW->QKPMNW",
             col, T2, X, X, Y, Y, T4)


def ins_up(row, T1, X, Y, T3):     # row (L,k,b,m,n,R); T1(d=Q, u=L); T3(u=R, d=W)
    return E("LkbmnR,QpqL,skpKr,sbqPv,tmrMw,tnvNx,RwxW->QKPMNW",
             row, T1, X, X, Y, Y, T3)


def ins_down(row, T1, X, Y, T3):   # row (L,k,b,m,n,R); T1(d=L, u=Q); T3(u=W, d=R)
    return E("LkbmnR,LpqQ,sKpkr,sPqbv,tMrmw,tNvnx,WwxR->QKPMNW",
             row, T1, X, X, Y, Y, T3)


def _nrm(x):
    return x / np.linalg.norm(x)


def _env(cfg):
    g = ci.generate(cfg)
    return {"C": g["C"], "T": g["T"]}, g["A"], g["B"]


def _expected_and_got(env, new, A, B, direction, x):
    y = O.OTHER[x]
    S = {"a": A, "b": B}
    C, T = env["C"], env["T"]
    nC, nT = new["C"], new["T"]
    if direction == "left":
        old = col_left(C[(x, 1)], T[(x, 1)], T[(y, 1)], C[(y, 4)])
        exp = ins_left(ins_left(old, T[(x, 2)], S[x], S[y], T[(y, 4)]), T[(y, 2)], S[y], S[x], T[(x, 4)])
        got = col_left(nC[(x, 1)], nT[(x, 1)], nT[(y, 1)], nC[(y, 4)])
    elif direction == "right":
        old = col_right(C[(x, 2)], T[(x, 3)], T[(y, 3)], C[(y, 3)])
        exp = ins_right(ins_right(old, T[(x, 2)], S[x], S[y], T[(y, 4)]), T[(y, 2)], S[y], S[x], T[(x, 4)])
        got = col_right(nC[(x, 2)], nT[(x, 3)], nT[(y, 3)], nC[(y, 3)])
    elif direction == "up":
        old = row_up(C[(x, 1)], T[(x, 2)], T[(y, 2)], C[(y, 2)])
        exp = ins_up(ins_up(old, T[(x, 1)], S[x], S[y], T[(y, 3)]), T[(y, 1)], S[y], S[x], T[(x, 3)])
        got = row_up(nC[(x, 1)], nT[(x, 2)], nT[(y, 2)], nC[(y, 2)])
    else:
        old = row_down(C[(x, 4)], T[(x, 4)], T[(y, 4)], C[(y, 3)])
        exp = ins_down(ins_down(old, T[(x, 1)], S[x], S[y], T[(y, 3)]), T[(y, 1)], S[y], S[x], T[(x, 3)])
        got = row_down(nC[(x, 4)], nT[(x, 4)], nT[(y, 4)], nC[(y, 3)])
    return _nrm(exp), _nrm(got)


@pytest.mark.parametrize("direction", ["left", "right", "up", "down"])
def test_full_move_without_truncation_is_exact(direction):
    """chi0 = 1 -> 4 -> 16 over a full move (both absorptions keep n = rows)."""
    cfg = ci.custom(2, 2, 16, chi0=1, seed_index=21)
    env, A, B = _env(cfg)
    new = O.move(env, A, B, direction, 16)
    for x in ("a", "b"):
        exp, got = _expected_and_got(env, new, A, B, direction, x)
        assert exp.shape == got.shape
        assert np.allclose(got, exp, atol=1e-12), np.abs(got - exp).max()


@pytest.mark.parametrize("direction", ["left", "right", "up", "down"])
def test_D1_move_is_exact(direction):
    cfg = ci.custom(2, 1, 3, seed_index=22)
    env, A, B = _env(cfg)
    new = O.move(env, A, B, direction, 3)
    for x in ("a", "b"):
        exp, got = _expected_and_got(env, new, A, B, direction, x)
        assert np.allclose(got, exp, atol=1e-12)


def test_single_absorption_chi0_4_to_16_is_exact():
    cfg = ci.custom(2, 2, 16, chi0=4, seed_index=23)
    env, A, B = _env(cfg)
    new, proj = O.column_absorption(env, A, B, 16)
    S = {"a": A, "b": B}
    C, T, nC, nT = env["C"], env["T"], new["C"], new["T"]
    for x in ("a", "b"):
        y = O.OTHER[x]
        v = proj[x + y]["v2"]
        assert v.shape[-1] == 16 and v.shape[0] * v.shape[1] == 16      # square: P = I
        old = col_left(C[(x, 1)], T[(x, 1)], T[(y, 1)], C[(y, 4)])
        exp = ins_left(old, T[(x, 2)], S[x], S[y], T[(y, 4)])
        got = col_left(nC[(y, 1)], nT[(y, 1)], nT[(x, 1)], nC[(x, 4)])
        assert np.allclose(_nrm(got), _nrm(exp), atol=1e-12)


def test_sequential_full_chi_prime_absorption_equals_reduced():
    """With chi' = chi0 D (v1 square) and chi'' = chi0 D^2 (exact reduced env), the
    sequential projectors equal the REDUCED ones, so the gauge-invariant
    contracted columns of one truncating absorption agree."""
    cfg = ci.custom(2, 2, 3, chi0=4, seed_index=24)
    env, A, B = _env(cfg)
    seq, _ = O.column_absorption(env, A, B, 3, chi_p=8, chi_pp=16, strategy="sequential")
    red, _ = O.column_absorption(env, A, B, 3, strategy="reduced")
    for x in ("a", "b"):
        y = O.OTHER[x]
        cs = col_left(seq["C"][(y, 1)], seq["T"][(y, 1)], seq["T"][(x, 1)], seq["C"][(x, 4)])
        cr = col_left(red["C"][(y, 1)], red["T"][(y, 1)], red["T"][(x, 1)], red["C"][(x, 4)])
        assert np.allclose(_nrm(cs), _nrm(cr), atol=1e-10)


def test_truncating_move_shapes_and_isometries():
    cfg = ci.CONFIGS["tiny"]
    env, A, B = _env(cfg)
    stats = []
    new = O.left_move(env, A, B, cfg.chi, stats=stats)
    for k, v in new["C"].items():
        assert v.shape == (8, 8)
        assert np.isclose(np.linalg.norm(v), 1.0) or k[1] in (2, 3)
    for k, v in new["T"].items():
        assert v.shape == (8, 2, 2, 8)
    assert all(np.isfinite(s["gap"]) or s["gap"] == np.inf for s in stats)


# ----------------------------------------------------------------------------------------
# convergence criterion (reading R22)
# ----------------------------------------------------------------------------------------
def test_corner_spectrum_closed_form():
    """diag(3, 2, 1) rotated by orthogonal matrices: spectrum (3, 2, 1) / 6."""
    rng = np.random.default_rng(5)
    Q1, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    Q2, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    C = Q1 @ np.diag([3.0, 2.0, 1.0]) @ Q2.T
    assert np.allclose(O.corner_spectrum(C), [0.5, 1 / 3, 1 / 6], atol=1e-14)


def test_spectra_distance_is_a_padded_l1_max():
    a = {("a", 1): np.array([0.6, 0.4]), ("b", 1): np.array([1.0])}
    b = {("a", 1): np.array([0.5, 0.3, 0.2]), ("b", 1): np.array([1.0])}
    assert O.spectra_distance(a, b) == pytest.approx(0.1 + 0.1 + 0.2)
    assert O.spectra_distance(a, a) == 0.0
    assert O.spectra_distance(a, b) == O.spectra_distance(b, a)


def test_converge_scalar_environment_in_one_sweep():
    """D = 1, chi = 1: every tensor is a scalar, every spectrum is (1) -- stationary from
    the first iteration (distance exactly 0)."""
    cfg = ci.custom(2, 1, 1, seed_index=41)
    g = ci.generate(cfg)
    _, it, delta = O.converge({"C": g["C"], "T": g["T"]}, g["A"], g["B"], 1, 1e-12, 10)
    assert it == 1 and delta == 0.0


def test_converge_iterations_monotone_in_tol():
    cfg = ci.CONFIGS["c2_dl"]
    g = ci.generate(cfg)
    env = {"C": g["C"], "T": g["T"]}
    _, it_loose, d_loose = O.converge(env, g["A"], g["B"], cfg.chi, 1e-4, 30)
    _, it_tight, d_tight = O.converge(env, g["A"], g["B"], cfg.chi, 1e-8, 30)
    assert it_loose <= it_tight
    assert d_tight < 1e-8 or it_tight == 30


# ----------------------------------------------------------------------------------------
# Reading R5 (which cut gets which projector; "P_ab and P_ba", "v_ba^1 contracts
# with boundary index of T_a^1 and virtual index of A"): a LOSSLESS TRUNCATION whose two cut
# types have different exact subspaces, so the assignment decides the result.
#   * Each site's down leg is rank one: X(s,u,l,d,r) = x(s,u,l,r) w_X(d), w_A != w_B.  The
#     legs crossing cut 'xy' (x above) -- T^1's boundary leg q and X's down legs (k, b) --
#     then carry vectors in q-space (x) w_X (x) w_X: exact rank chi0 of chi0 D^2 rows.
#   * The top edge above x is consistent with the lattice (the site above x is y):
#     T_x^2(l,k,b,r) = t(l,r) w_Y(k) w_Y(b).
# With chi = chi0 every truncation keeps chi0 of chi0 D^2 rows and is exact for the right
# assignment: the new column contracted along its bonds equals old column (x) inserted
# column.  Swapping V_ab <-> V_ba (same shapes, so only the values can tell) projects X's
# legs onto w_Y (x) w_Y and the column changes.
# ----------------------------------------------------------------------------------------
def _r5_case(seed=77, d=2, D=2, chi0=2):
    rng = np.random.default_rng(seed)
    w = {"a": rng.standard_normal(D), "b": rng.standard_normal(D)}
    site = {}
    for x in ("a", "b"):
        core = rng.standard_normal((d, D, D, D))                     # (s, u, l, r)
        site[x] = np.einsum("sulr,d->suldr", core, w[x])
        site[x] /= np.linalg.norm(site[x])
    cfg = ci.custom(d, D, chi0, chi0=chi0, seed_index=78)
    g = ci.generate(cfg)
    C, T = dict(g["C"]), dict(g["T"])
    for x in ("a", "b"):
        y = O.OTHER[x]
        t = rng.standard_normal((chi0, chi0))
        T[(x, 2)] = np.einsum("lr,k,b->lkbr", t, w[y], w[y])
        T[(x, 2)] /= np.linalg.norm(T[(x, 2)])
    return {"C": C, "T": T}, site["a"], site["b"], chi0


@pytest.mark.parametrize("strategy", ["sequential", "reduced"])
def test_r5_cut_assignment_is_exact_on_a_lossless_truncation(strategy):
    env, A, B, chi = _r5_case()
    S = {"a": A, "b": B}
    stats = []
    new, proj = O.column_absorption(env, A, B, chi, chi, chi, strategy=strategy, stats=stats)
    C, T, nC, nT = env["C"], env["T"], new["C"], new["T"]
    for x in ("a", "b"):
        y = O.OTHER[x]
        V = proj[x + y]["V"] if strategy == "reduced" else O.compose_isometry(proj[x + y]["v1"], proj[x + y]["v2"])
        assert V.shape == (chi, 2, 2, chi)   # keeps chi of chi D^2 = 4 chi rows: a real truncation
        old = col_left(C[(x, 1)], T[(x, 1)], T[(y, 1)], C[(y, 4)])
        exp = ins_left(old, T[(x, 2)], S[x], S[y], T[(y, 4)])
        got = col_left(nC[(y, 1)], nT[(y, 1)], nT[(x, 1)], nC[(x, 4)])
        assert np.allclose(_nrm(got), _nrm(exp), atol=1e-12), np.abs(_nrm(got) - _nrm(exp)).max()


@pytest.mark.parametrize("strategy", ["sequential", "reduced"])
def test_r5_swapped_cut_assignment_fails(strategy):
    """The deliberately mis-assigned projectors (V_ab at the 'ba' cuts and vice versa) break
    the same identity: the pin above cannot pass with the wrong reading."""
    env, A, B, chi = _r5_case()
    S = {"a": A, "b": B}
    own = O._cut_projectors(env, A, B, chi, chi, chi, strategy, None)
    swapped = {"ab": own["ba"], "ba": own["ab"]}
    new, _ = O.column_absorption(env, A, B, chi, chi, chi, strategy=strategy, projectors=swapped)
    C, T, nC, nT = env["C"], env["T"], new["C"], new["T"]
    worst = 0.0
    for x in ("a", "b"):
        y = O.OTHER[x]
        exp = ins_left(col_left(C[(x, 1)], T[(x, 1)], T[(y, 1)], C[(y, 4)]), T[(x, 2)], S[x], S[y], T[(y, 4)])
        got = col_left(nC[(y, 1)], nT[(y, 1)], nT[(x, 1)], nC[(x, 4)])
        worst = max(worst, min(np.abs(_nrm(got) - _nrm(exp)).max(), np.abs(_nrm(got) + _nrm(exp)).max()))
    assert worst > 1e-3, worst

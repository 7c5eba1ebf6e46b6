"""Pins of the oracle's closures: 2x2 norm, bond rho / energy, double layer
(SURVEY 8(c) rows '2x2 norm', 'Double layer', 'rho and energy')."""
import json
import os

import numpy as np
import pytest

import ctm_inputs as ci
from oracle import ctm_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _env(cfg):
    g = ci.generate(cfg)
    return {"C": g["C"], "T": g["T"]}, g["A"], g["B"]


def _fused_site(X):
    D = X.shape[1]
    a = np.einsum("sabcd,sefgh->aebfcgdh", X, X)
    return a.reshape(D * D, D * D, D * D, D * D)


def _fused_T(t):
    c0, D, _, c1 = t.shape
    return t.reshape(c0, D * D, c1)


def _rows_top(C, T):
    # top row C_a^1(d=x, r=y) T_a^2(l=y, e, r=Y) T_b^2(l=Y, i, r=z) C_b^2(l=z, d=w) -> (x, e, i, w)
    R = np.einsum("xy,yeY->xeY", C[("a", 1)], T[("a", 2)])
    R = np.einsum("xeY,Yiz->xeiz", R, T[("b", 2)])
    return np.einsum("xeiz,zw->xeiw", R, C[("b", 2)])


def norm_2x2_fused(env, A, B):
    """Independent formulation: fused double-layer tensors a = sum_s A A* (Fig 1(b))
    with D^2 legs, contracted row by row (transfer-matrix order) instead of by corners."""
    C, T = env["C"], {k: _fused_T(v) for k, v in env["T"].items()}
    a, b = _fused_site(A), _fused_site(B)                      # (u, l, d, r)
    R = _rows_top(C, T)                                         # (x, e, i, w)
    # row 1: T_a^1(d=X, f, u=x)  a(e,f,g,h)  b(i,h,j,k)  T_b^3(u=w, k, d=W)
    R = np.einsum("xeiw,Xfx->eiwXf", R, T[("a", 1)])
    R = np.einsum("eiwXf,efgh->iwXgh", R, a)
    R = np.einsum("iwXgh,ihjk->wXgjk", R, b)
    R = np.einsum("wXgjk,wkW->XgjW", R, T[("b", 3)])
    # row 2: T_b^1(d=q, l, u=X)  b(g,l,m,n)  a(j,n,o,p)  T_a^3(u=W, p, d=v)
    R = np.einsum("XgjW,qlX->gjWql", R, T[("b", 1)])
    R = np.einsum("gjWql,glmn->jWqmn", R, b)
    R = np.einsum("jWqmn,jnop->Wqmop", R, a)
    R = np.einsum("Wqmop,Wpv->qmov", R, T[("a", 3)])
    # bottom: C_b^4(r=Z, u=q) T_b^4(r=U, m, l=Z) T_a^4(r=V, o, l=U) C_a^3(u=v, l=V)
    R = np.einsum("qmov,Zq->movZ", R, C[("b", 4)])
    R = np.einsum("movZ,UmZ->ovU", R, T[("b", 4)])
    R = np.einsum("ovU,VoU->vV", R, T[("a", 4)])
    return float(np.einsum("vV,vV->", R, C[("a", 3)]))


@pytest.mark.parametrize("D,chi,seed", [(2, 4, 31), (2, 8, 32), (3, 3, 33)])
def test_norm_two_independent_orders(D, chi, seed):
    env, A, B = _env(ci.custom(2, D, chi, seed_index=seed))
    n1 = O.norm_2x2(env, A, B)
    n2 = norm_2x2_fused(env, A, B)
    assert np.isclose(n1, n2, rtol=1e-11, atol=0)


def test_norm_D1_chi1_closed_form():
    env, A, B = _env(ci.custom(2, 1, 1, seed_index=34))
    # every env tensor is a +-1 scalar after Frobenius normalisation; unit A, B
    labels = [("C", "a", 1), ("T", "a", 2), ("T", "b", 2), ("C", "b", 2), ("T", "b", 3), ("T", "a", 3),
              ("C", "a", 3), ("T", "a", 4), ("T", "b", 4), ("C", "b", 4), ("T", "b", 1), ("T", "a", 1)]
    prod = np.prod([env[k][(x, n)].ravel()[0] for k, x, n in labels])
    assert np.isclose(abs(prod), 1.0)
    assert np.isclose(O.norm_2x2(env, A, B), prod * np.sum(A ** 2) ** 2 * np.sum(B ** 2) ** 2, rtol=1e-14)


def test_norm_homogeneity():
    env, A, B = _env(ci.custom(2, 2, 4, seed_index=35))
    n = O.norm_2x2(env, A, B)
    assert np.isclose(O.norm_2x2(env, 1.3 * A, B), 1.3 ** 4 * n, rtol=1e-12)
    assert np.isclose(O.norm_2x2(env, A, 0.7 * B), 0.7 ** 4 * n, rtol=1e-12)


def test_double_layer_bra_ket_symmetric():
    rng = np.random.default_rng(36)
    A = rng.standard_normal((2, 3, 3, 3, 3))
    a = O.double_layer(A)
    # swap every (ket, bra) pair: (uk,ub,lk,lb,dk,db,rk,rb) -> (ub,uk,...)
    assert np.allclose(a, a.transpose(1, 0, 3, 2, 5, 4, 7, 6), atol=1e-15)
    # elementwise loop oracle on a few entries
    for idx in [(0, 1, 2, 0, 1, 1, 2, 0), (2, 2, 0, 1, 0, 2, 1, 1)]:
        want = sum(A[s, idx[0], idx[2], idx[4], idx[6]] * A[s, idx[1], idx[3], idx[5], idx[7]] for s in range(2))
        assert np.isclose(a[idx], want)


def test_heisenberg_operator_golden():
    g = json.load(open(os.path.join(GOLD, "heisenberg_bond.json")))
    h = ci.heisenberg_h()
    H = h.reshape(4, 4)
    assert np.allclose(H, np.array(g["h_matrix_basis_uu_ud_du_dd"]), atol=1e-15)
    assert np.allclose(np.linalg.eigvalsh(H), g["spectrum"], atol=1e-14)
    assert np.isclose(np.trace(H), g["trace"])


@pytest.mark.parametrize("bond", ["H", "V"])
def test_energy_D1_closed_form(bond):
    env, A, B = _env(ci.custom(2, 1, 3, seed_index=37))
    h = ci.heisenberg_h()
    e, m = O.bond_energy(env, A, B, h, bond)
    a, b = A.ravel(), B.ravel()
    ab = np.kron(a, b)
    want = ab @ h.reshape(4, 4) @ ab / (a @ a) / (b @ b)
    assert np.isclose(e, want, rtol=1e-12)
    assert np.isclose(np.trace(m), 1.0)
    assert -0.75 - 1e-12 <= e <= 0.25 + 1e-12


@pytest.mark.parametrize("bond", ["H", "V"])
def test_rho_product_state_closed_form(bond):
    """Sites rank-1 in the virtual legs, A = phi(s) a(u) b(l) c(d) e(r): the state is a
    product state, so for ANY environment rho factorises into phi_A phi_A^T (x) phi_B phi_B^T."""
    rng = np.random.default_rng(38)
    D = 2
    env, _, _ = _env(ci.custom(2, D, 4, seed_index=38))
    def prod_site():
        vs = [rng.standard_normal(D) for _ in range(4)]
        phi = rng.standard_normal(2)
        return np.einsum("s,u,l,d,r->suldr", phi, *vs), phi
    A, pa = prod_site()
    B, pb = prod_site()
    h = ci.heisenberg_h()
    e, m = O.bond_energy(env, A, B, h, bond)
    ab = np.kron(pa, pb) / np.linalg.norm(pa) / np.linalg.norm(pb)
    assert np.allclose(m, np.outer(ab, ab), atol=1e-12)
    assert np.isclose(e, ab @ h.reshape(4, 4) @ ab, rtol=1e-11)


def test_rho_trace_is_window_norm():
    """Tr rho_H equals the fused-double-layer contraction of the 2x1 window."""
    env, A, B = _env(ci.custom(2, 2, 4, seed_index=39))
    rho = O.bond_rho(env, A, B, "H")
    tr = np.einsum("abab->", rho)
    C, T = env["C"], {k: _fused_T(v) for k, v in env["T"].items()}
    a, b = _fused_site(A), _fused_site(B)
    R = _rows_top(C, T)                                         # (x, e, i, w)
    R = np.einsum("xeiw,Xfx->eiwXf", R, T[("a", 1)])
    R = np.einsum("eiwXf,efgh->iwXgh", R, a)
    R = np.einsum("iwXgh,ihjk->wXgjk", R, b)
    R = np.einsum("wXgjk,wkW->XgjW", R, T[("b", 3)])            # (X, g=a's d, j=b's d, W)
    # bottom: C_a^4(r=Z, u=X) T_a^4(r=U, g, l=Z) T_b^4(r=V, j, l=U) C_b^3(u=W, l=V)
    R = np.einsum("XgjW,ZX->gjWZ", R, C[("a", 4)])
    R = np.einsum("gjWZ,UgZ->jWU", R, T[("a", 4)])
    R = np.einsum("jWU,VjU->WV", R, T[("b", 4)])
    want = np.einsum("WV,WV->", R, C[("b", 3)])
    assert np.isclose(tr, want, rtol=1e-11)


# ----------------------------------------------------------------------------------------
# single-site spins and staggered magnetisation (reading R23)
# ----------------------------------------------------------------------------------------
def _spin(phi):
    phi = phi / np.linalg.norm(phi)
    sx = np.array([[0.0, 0.5], [0.5, 0.0]])
    sz = np.array([[0.5, 0.0], [0.0, -0.5]])
    return phi @ sx @ phi, phi @ sz @ phi


def test_site_spins_product_state_closed_form():
    """A = phi(s) a(u) b(l) c(d) e(r): for ANY environment <S>_A = phi^T S phi / |phi|^2."""
    rng = np.random.default_rng(40)
    D = 2
    env, _, _ = _env(ci.custom(2, D, 4, seed_index=40))

    def prod_site():
        vs = [rng.standard_normal(D) for _ in range(4)]
        phi = rng.standard_normal(2)
        return np.einsum("s,u,l,d,r->suldr", phi, *vs), phi
    A, pa = prod_site()
    B, pb = prod_site()
    (xa, za), (xb, zb) = O.site_spins(env, A, B)
    assert np.allclose((xa, za), _spin(pa), atol=1e-12)
    assert np.allclose((xb, zb), _spin(pb), atol=1e-12)
    want = 0.5 * (np.hypot(*_spin(pa)) + np.hypot(*_spin(pb)))
    assert np.isclose(O.staggered_magnetization(env, A, B), want, rtol=1e-12)


def test_site_spins_neel_state():
    """Neel product state (A up, B down along z): <S^z> = +1/2, -1/2, m_s = 1/2."""
    env, _, _ = _env(ci.custom(2, 1, 3, seed_index=42))
    A = np.array([1.0, 0.0]).reshape(2, 1, 1, 1, 1)
    B = np.array([0.0, 1.0]).reshape(2, 1, 1, 1, 1)
    (xa, za), (xb, zb) = O.site_spins(env, A, B)
    assert np.allclose((xa, za, xb, zb), (0.0, 0.5, 0.0, -0.5), atol=1e-14)
    assert np.isclose(O.staggered_magnetization(env, A, B), 0.5)


def test_site_spins_bounded_for_a_positive_environment():
    """With the partial-trace (positive) start the window rho is a density matrix, so
    |<S>| <= 1/2 (a Gaussian environment is not positive and carries no such bound)."""
    cfg = ci.custom(2, 2, 4, seed_index=43)
    g = ci.generate(cfg, "double_layer")
    for x, z in O.site_spins({"C": g["C"], "T": g["T"]}, g["A"], g["B"]):
        assert np.hypot(x, z) <= 0.5 + 1e-12


# ----------------------------------------------------------------------------------------
# reduced_env_exact (Fig 3(a,b)) closed with the rest of its window
# ----------------------------------------------------------------------------------------
def _window_3x3_fused(C1, T2, C2, T1, X, Xb, T3, C4, T4, C3):
    """<psi|psi> of the 3x3 window  C1 T2 C2 / T1 X T3 / C4 T4 C3  (clockwise storage),
    formulated independently of reduced_env_exact: fused double layer a = sum_s X X* with
    D^2 legs (ket != bra allowed), fused edges, contracted row by row."""
    D = X.shape[1]
    a = np.einsum("sabcd,sefgh->aebfcgdh", X, Xb).reshape(D * D, D * D, D * D, D * D)   # (u, l, d, r)
    f = lambda t: t.reshape(t.shape[0], D * D, t.shape[3])
    # top row: C1(d=i, r=p) T2(l=p, j, r=q) C2(l=q, d=k) -> (i, j, k)
    R = np.einsum("ip,pjq->ijq", C1, f(T2))
    R = np.einsum("ijq,qk->ijk", R, C2)
    # middle row: T1(d=I, l, u=i)  a(j, l, J, r)  T3(u=k, r, d=K)
    R = np.einsum("ijk,Ili->jkIl", R, f(T1))
    R = np.einsum("jkIl,jlJr->kIJr", R, a)
    R = np.einsum("kIJr,krK->IJK", R, f(T3))
    # bottom row: C4(r=m, u=I)  T4(r=n, J, l=m)  C3(u=K, l=n)
    R = np.einsum("IJK,mI->JKm", R, C4)
    R = np.einsum("JKm,nJm->Kn", R, f(T4))
    return float(np.einsum("Kn,Kn->", R, C3))


@pytest.mark.parametrize("D,chi,seed", [(2, 4, 51), (3, 5, 52)])
def test_reduced_env_exact_closes_to_the_window_norm(D, chi, seed):
    """M_exact(q, k_d, b_d, q') closed with the bottom row C^4 T^4 C^3 equals the 3x3 window
    norm computed in the fused row-transfer order; ket != bra catches ket/bra mix-ups, random
    rectangular-free extents catch transposed boundary legs."""
    rng = np.random.default_rng(seed)
    d = 2
    C1, C2, C3, C4 = (rng.standard_normal((chi, chi)) for _ in range(4))
    T1, T2, T3, T4 = (rng.standard_normal((chi, D, D, chi)) for _ in range(4))
    X = rng.standard_normal((d, D, D, D, D))
    Xb = rng.standard_normal((d, D, D, D, D))
    M = O.reduced_env_exact(C1, T2, C2, T1, X, Xb, T3)
    # bottom row: C4 (r=m, u=q), T4 (r=n, k, b, l=m), C3 (u=q', l=n)
    closed = np.einsum("qkbz,mq,nkbm,zn->", M, C4, T4, C3)
    want = _window_3x3_fused(C1, T2, C2, T1, X, Xb, T3, C4, T4, C3)
    assert closed == pytest.approx(want, rel=1e-11)
    # the closure is not blind to a ket/bra exchange of the down legs
    closed_swapped = np.einsum("qbkz,mq,nkbm,zn->", M, C4, T4, C3)
    assert abs(closed_swapped - want) > 1e-6 * abs(want)

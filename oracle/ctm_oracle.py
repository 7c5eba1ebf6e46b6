"""CPU float64 oracle for the CTMRG move of arXiv 2306.08212 (Lan & Evenbly).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module.  The
product path (`paper_2306_08212_b200/`) never imports it and shares no code with it;
both sides only share the seeded input generator `ctm_inputs.py`.

Every function follows the paper step by step (PAPER.md = "P:Lnn") in the readings
fixed by SURVEY.md sections 0 and 8(c) (listed again in DESIGN.md "Readings").  Each
pairwise contraction is one `numpy.einsum` of two operands (a BLAS-backed library
primitive); SVDs are LAPACK (`numpy.linalg.svd`).  No blocking, fusion or reordering
beyond the order the paper/survey states.

Conventions:
  * site tensor X (s,u,l,d,r); bra layer X* = X (real configs, reading R15);
  * clockwise storage: T^1 (d,k,b,u), T^2 (l,k,b,r), T^3 (u,k,b,d), T^4 (r,k,b,l),
    C^1 (d,r), C^2 (l,d), C^3 (u,l), C^4 (r,u); k/b = ket/bra legs facing the bulk;
  * env = {"C": {(x,k): arr}, "T": {(x,k): arr}}, x in ("a","b"), k in 1..4;
  * the 2x2 patch (Fig 1(d)):
        C_a^1  T_a^2  T_b^2  C_b^2
        T_a^1    A      B    T_b^3
        T_b^1    B      A    T_a^3
        C_b^4  T_b^4  T_a^4  C_a^3

Pins: tests/test_oracle_*.py (run with -m "not gpu").  Functions without a pin other
than GPU parity are marked "parity unpinned" below and in DESIGN.md.
"""
from __future__ import annotations

import numpy as np

SUBS = ("a", "b")
OTHER = {"a": "b", "b": "a"}


def _c(spec: str, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """One pairwise contraction (library primitive: einsum -> tensordot/BLAS)."""
    return np.einsum(spec, x, y, optimize=True)


def frob_normalise(x: np.ndarray) -> np.ndarray:
    """N[x] = x / ||x||_F  (environment normalisation, reading R13; P:L43 is silent)."""
    return x / np.linalg.norm(x)


# ----------------------------------------------------------------------------------
# Truncated SVD and the two-stage isometry (appendix)
# ----------------------------------------------------------------------------------

def sign_fix(U: np.ndarray) -> np.ndarray:
    """Sign rule: in each column the entry of largest
    |.| is made positive; ties go to the lowest row index (argmax returns the first)."""
    if U.size == 0:
        return U
    idx = np.argmax(np.abs(U), axis=0)
    s = np.sign(U[idx, np.arange(U.shape[1])])
    s[s == 0] = 1.0
    return U * s[None, :]


def left_singular(mat: np.ndarray, n: int, stats: list | None = None) -> np.ndarray:
    """First n left singular vectors of `mat` ("the unitary matrix U is reshaped ...
    truncation applied corresponding to the largest chi singular values").

    n may exceed min(rows, cols) (reading R11): then the columns come from the full U;
    they are meaningful only when n == rows (square orthogonal U, projector = I)."""
    rows, cols = mat.shape
    assert 1 <= n <= rows, (n, rows)
    full = n > min(rows, cols)
    U, S, _ = np.linalg.svd(mat, full_matrices=full)
    if stats is not None:
        kept = min(n, S.size)
        gap = S[kept - 1] / S[kept] if kept < S.size and S[kept] > 0 else np.inf
        stats.append({"shape": (rows, cols), "n": n, "sigma_first": float(S[0]) if S.size else 0.0,
                      "sigma_last_kept": float(S[kept - 1]) if kept else 0.0, "gap": float(gap),
                      "rank_deficient_null_columns": bool(n > S.size and n < rows)})
    return sign_fix(U[:, :n])


def ts_isometry(Q: np.ndarray, c1: int, c2: int, stats: list | None = None):
    """Two-stage isometry TS(Q; c1, c2) of SURVEY 0 ("we reshape it to matrix
    of dimension chi D x chi D ... U_d^1 reshaped to v^1 ... truncating according to the
    largest chi' singular values ... contract v^1 with environments ... additional SVD on
    (chi D, chi) matrix to obtain U_d^2, which serves as v^2").

    Q(p,k,b,q): p boundary leg, k ket leg, b bra leg (the cut legs), q the far leg.
    Returns v1 (p,k,n1) and v2 (n1,b,n2), n1 = min(c1, p*k), n2 = min(c2, n1*b)."""
    P, K, B, F = Q.shape
    n1 = min(c1, P * K)
    v1 = left_singular(Q.reshape(P * K, B * F), n1, stats).reshape(P, K, n1)
    Q2 = _c("pka,pkbq->abq", v1, Q)                       # v^1 contracted into the env
    n2 = min(c2, n1 * B)
    v2 = left_singular(Q2.reshape(n1 * B, F), n2, stats).reshape(n1, B, n2)
    return v1, v2


def compose_isometry(v1: np.ndarray, v2: np.ndarray) -> np.ndarray:
    """V(p,k,b,beta) = sum_alpha v1(p,k,alpha) v2(alpha,b,beta) (v_ba ~ v^1 v^2)."""
    return _c("pka,abz->pkbz", v1, v2)


def one_shot_isometry(M: np.ndarray, chi: int, stats: list | None = None) -> np.ndarray:
    """REDUCED/STANDARD projector ("chi D^2 x chi in FIG 3(b)"):
    V = first chi left singular vectors of M grouped as (p,k,b) x (rest).
    Returns V(p,k,b,n), n = min(chi, p*k*b)."""
    P, K, B = M.shape[:3]
    rest = int(np.prod(M.shape[3:]))
    n = min(chi, P * K * B)
    return left_singular(M.reshape(P * K * B, rest), n, stats).reshape(P, K, B, n)


# ----------------------------------------------------------------------------------
# Sequential absorb/truncate chain (rows a6-a8) and corner growth (row a9)
# ----------------------------------------------------------------------------------

def orient_left(X: np.ndarray) -> np.ndarray:
    """Site X (s,u,l,d,r) seen from a LEFT edge T^1 stored (d,k,b,u):
    (s, in=d, face=l, out=u, far=r)."""
    return X.transpose(0, 3, 2, 1, 4)


def orient_top(X: np.ndarray) -> np.ndarray:
    """Site X (s,u,l,d,r) seen from a TOP edge T^2 stored (l,k,b,r):
    (s, in=l, face=u, out=r, far=d)."""
    return X.transpose(0, 2, 1, 4, 3)


def absorb_truncate(T, Xo, Xbo, v1_in, v2_in, v1_out, v2_out):
    """Sequential-order edge update (Fig 4(b)):
    ket absorption, truncation with v^1, bra absorption, truncation with v^2.

    T (p, kf, bf, q): p = 'in' boundary leg, (kf,bf) face legs, q = 'out' boundary leg.
    Xo, Xbo (s, in, face, out, far) ket / bra site in chain orientation.
    v1_in (p, k_in, alpha), v2_in (alpha, b_in, o1): isometry of the cut on the 'in' side;
    v1_out (q, k_out, beta), v2_out (beta, b_out, o2): isometry of the cut on the 'out' side.
    Returns T'(o1, k_far, b_far, o2)."""
    # S1: "v^1 contracts with boundary index of T ..."       K = chi
    X1 = _c("pia,pfgq->aifgq", v1_in, T)
    # S2: "... and virtual index of A" -> absorb the ket site over (in, face)   K = D^2
    X2 = _c("aifgq,sifoz->agqsoz", X1, Xo)
    # S3: truncate the 'out' cut's (boundary, ket) pair with v^1_out          K = chi D
    X3 = _c("agqsoz,qob->agszb", X2, v1_out)
    # S4: "v^2 contracts with boundary index ..." : v^2_in over alpha          K = chi'
    X4 = _c("agszb,ajc->gszbjc", X3, v2_in)
    # S5: "... and virtual index of A^dagger": bra site over (s, face, in)     K = d D^2
    X5 = _c("gszbjc,sjgyw->zbcyw", X4, Xbo)
    # S6: truncate the 'out' cut's (boundary', bra) pair with v^2_out          K = chi' D
    return _c("zbcyw,byd->czwd", X5, v2_out)


def absorb_one_shot(T, Xo, Xbo, V_in, V_out):
    """STANDARD/REDUCED edge update with 4-leg isometries (Fig 2(b)):
    T'(o1,kz,bz,o2) = sum V_in(p,ki,bi,o1) T(p,kf,bf,q) X(s,ki,kf,ko,kz) X*(s,bi,bf,bo,bz)
    V_out(q,ko,bo,o2).  Cost chi^3 D^4 or more (the cost the paper removes)."""
    Y = _c("pjko,pfgq->jkofgq", V_in, T)                # (ki, bi, o1, kf, bf, q)
    Y = _c("jkofgq,sjfaz->kogqsaz", Y, Xo)               # over ki, kf
    Y = _c("kogqsaz,skgbw->oqazbw", Y, Xbo)              # over bi, bf, s
    return _c("oqazbw,qabd->ozwd", Y, V_out)             # over q, ko, bo


def corner_top_left(C1, T2, v1, v2):
    """Corner growth C^1' = ((C^1 v^1) T^2) v^2 ("(C_a^1, T_a^2) -> C_b^1"; Fig 4(b);
    SURVEY row a9).  C^1 stored (d,r); T^2 stored (l,k,b,r); v1 (d-bond, k, alpha),
    v2 (alpha, b, o).  Returns C^1'(o, r') in storage (d, r)."""
    Y1 = _c("xp,xka->pka", C1, v1)
    Y2 = _c("pka,pkbr->abr", Y1, T2)
    return _c("abr,abo->or", Y2, v2)


def corner_bottom_left(C4, T4, v1, v2):
    """Corner growth C^4' ("(C_b^4, T_b^4) -> C_a^4"; SURVEY row a9 mirrored).
    C^4 stored (r,u); T^4 stored (r,k,b,l); v1 (u-bond, k, alpha), v2 (alpha, b, o).
    Returns C^4'(r', o) in storage (r, u)."""
    Y1 = _c("px,xka->pka", C4, v1)                       # C4[p=r, x=u]
    Y2 = _c("pka,rkbp->abr", Y1, T4)                     # T4[r', k, b, l=p]
    return _c("abr,abo->ro", Y2, v2)


def corner_top_left_one_shot(C1, T2, V):
    return _c("xkbr,xkbo->or", _c("xp,pkbr->xkbr", C1, T2), V)


def corner_bottom_left_one_shot(C4, T4, V):
    return _c("xkbr,xkbo->ro", _c("px,rkbp->xkbr", C4, T4), V)


# ----------------------------------------------------------------------------------
# Reduced environment (Fig 3; appendix, rows a1-a4)
# ----------------------------------------------------------------------------------

def side_products(C1, T1, C2, T3):
    """Row a1: Q_l(p,k,b,q) = C^1 . T^1 (p = C^1's r leg, q = T^1's d leg) and
    Q_r(p,k,b,q) = C^2 . T^3 (p = C^2's l leg, q = T^3's d leg).
    'by only considering the environment tensors {C_a^1, T_a^1}'."""
    Ql = _c("xp,qkbx->pkbq", C1, T1)      # C1 (d=x, r=p);  T1 (d=q, k, b, u=x)
    Qr = _c("px,xkbq->pkbq", C2, T3)      # C2 (l=p, d=x);  T3 (u=x, k, b, d=q)
    return Ql, Qr


def reduced_env_approx(C1, T2, C2, T1, X, Xb, T3, chi_pp: int, stats: list | None = None,
                       isos=None):
    """Approximated reduced environment M = C'^1 T'^2 C'^2 ("{C'_b^1, T'_b^2, C'_b^2}
    can be obtained ... at the cost of O(chi^3 D^3) (Appendix)", Fig 3(c)).

    Returns (M, (vl1, vl2, vr1, vr2)); M (q, k_d, b_d, q') with q = T^1's d leg,
    (k_d, b_d) = X's down legs, q' = T^3's d leg.  `isos` injects the side isometries."""
    Ql, Qr = side_products(C1, T1, C2, T3)                           # a1
    if isos is None:                                                 # a2
        vl1, vl2 = ts_isometry(Ql, chi_pp, chi_pp, stats)
        vr1, vr2 = ts_isometry(Qr, chi_pp, chi_pp, stats)
    else:
        vl1, vl2, vr1, vr2 = isos
    Cl = _c("pkbq,pka->abq", Ql, vl1)                                # a4: C'(q, lam)
    Cl = _c("abq,abl->ql", Cl, vl2)
    Cr = _c("pkbq,pka->abq", Qr, vr1)                                # a4: C''(rho, q')
    Cr = _c("abq,abr->rq", Cr, vr2)
    Tp = absorb_truncate(T2, orient_top(X), orient_top(Xb), vl1, vl2, vr1, vr2)   # a3
    M = _c("ql,lkbr->qkbr", Cl, Tp)                                  # a4
    M = _c("qkbr,rz->qkbz", M, Cr)
    return M, (vl1, vl2, vr1, vr2)


def reduced_env_exact(C1, T2, C2, T1, X, Xb, T3):
    """Exact reduced environment (Fig 3(a,b)):
    M(q,kd,bd,q') = sum C^1 T^2 C^2 T^1 X X* T^3, the right half replaced by {C^2,T^3}
    ('the isometry v is from right move, and won't be used in this step')."""
    R = _c("xp,pkbz->xkbz", C1, T2)                  # C1 (d=x, r=p), T2 (l=p, ku, bu, r=z)
    R = _c("xkbz,zy->xkby", R, C2)                   # C2 (l=z, d=y)
    R = _c("xkby,qlmx->kbyqlm", R, T1)               # T1 (d=q, kl, bl, u=x)
    R = _c("kbyqlm,skldr->bymqsdr", R, X)            # X (s, u=k, l, d, r) over ku, kl
    R = _c("bymqsdr,sbmew->yqdrew", R, Xb)           # X* (s, u=b, l=m, d=e, r=w) over s,bu,bl
    return _c("yqdrew,yrwz->qdez", R, T3)            # T3 (u=y, kr, br, d=z)


def half_network_standard(C1x, T2x, T2y, C2y, T1x, X, Xb, Y, Yb, T3y):
    """STANDARD sub-network (P:L46, P:L53 '8 individual tensors', Fig 2(c)): upper half
    of the 2x2 patch, open at the bottom:
            C_x^1  T_x^2  T_y^2  C_y^2
            T_x^1    X      Y    T_y^3
    Returns M_std(q, kX, bX, kY, bY, q') with q = T_x^1's d leg, q' = T_y^3's d leg."""
    # bonds: C1x(d=e, r=f) T2x(l=f, ku=g, bu=h, r=i) T2y(l=i, ku=j, bu=k, r=l) C2y(l=l, d=m)
    #        T3y(u=m, kr=n, br=o, d=Q) T1x(d=P, kl=p, bl=q, u=e)
    #        X(s, u=g, l=p, d=K, r=r) X*(s, u=h, l=q, d=B, r=w)
    #        Y(s, u=j, l=r, d=L, r=n) Y*(s, u=k, l=w, d=E, r=o)
    Lh = _c("ef,Ppqe->fPpq", C1x, T1x)
    Lh = _c("fPpq,fghi->Ppqghi", Lh, T2x)
    Lh = _c("Ppqghi,sgpKr->PqhisKr", Lh, X)
    Lh = _c("PqhisKr,shqBw->PiKrBw", Lh, Xb)
    Rh = _c("ijkl,lm->ijkm", T2y, C2y)
    Rh = _c("ijkm,mnoQ->ijknoQ", Rh, T3y)
    Rh = _c("ijknoQ,sjrLn->ikoQsrL", Rh, Y)
    Rh = _c("ikoQsrL,skwEo->iQrLwE", Rh, Yb)
    return _c("PiKrBw,iQrLwE->PKBLEQ", Lh, Rh)


# ----------------------------------------------------------------------------------
# Column absorption and moves
# ----------------------------------------------------------------------------------

def _cut_projectors(env, A, B, chi, chi_p, chi_pp, strategy, stats, renv_isos=None):
    """Projectors of the two cut types.  Cut 'xy' has site x above it; V_xy comes from
    M_xy built from x-labelled tensors (reading R5)."""
    C, T = env["C"], env["T"]
    site = {"a": A, "b": B}
    out = {}
    for x in SUBS:
        y = OTHER[x]
        X = site[x]
        if strategy == "sequential":
            inj = None if renv_isos is None else renv_isos.get(x)
            M, side = reduced_env_approx(C[(x, 1)], T[(x, 2)], C[(x, 2)], T[(x, 1)], X, X,
                                         T[(x, 3)], chi_pp, stats, isos=inj)
            v1, v2 = ts_isometry(M, chi_p, chi, stats)
            out[x + y] = {"M": M, "v1": v1, "v2": v2, "side": side}
        elif strategy == "reduced":
            M = reduced_env_exact(C[(x, 1)], T[(x, 2)], C[(x, 2)], T[(x, 1)], X, X, T[(x, 3)])
            out[x + y] = {"M": M, "V": one_shot_isometry(M, chi, stats)}
        elif strategy == "standard":
            Y = site[y]
            M = half_network_standard(C[(x, 1)], T[(x, 2)], T[(y, 2)], C[(y, 2)], T[(x, 1)],
                                      X, X, Y, Y, T[(y, 3)])
            out[x + y] = {"M": M, "V": one_shot_isometry(M, chi, stats)}
        else:
            raise ValueError(strategy)
    return out


def column_absorption(env, A, B, chi, chi_p=None, chi_pp=None, strategy="sequential",
                      stats=None, projectors=None, renv_isos=None, normalise=True):
    """One column absorption: insert {T^2, X, Y, T^4}, absorb, truncate.
    Both row-parity windows are updated from one snapshot (reading R3).  For the window
    whose absorbed column has site x on top and y below it:
        C_y^1 <- N[C_x^1 T_x^2 V_yx]            (cut above x: 'yx')
        T_y^1 <- N[V_xy T_x^1 X X* V_yx]        (in = cut below x, out = cut above x)
        C_x^4 <- N[V_yx C_y^4 T_y^4]            (cut above the corner row, below y: 'yx')
    i.e. for x = a: C_b^1 <- C_a^1 T_a^2 V_ba, T_b^1 <- V_ba T_a^1 A A* V_ab,
    C_a^4 <- V_ba C_b^4 T_b^4 -- the output set {C_b^1, T_b^1, T_a^1, C_a^4} of P:L43.
    `projectors` injects {'ab': {...}, 'ba': {...}} (identical-isometry tests).
    Returns (new_env, projectors)."""
    chi_p = chi if chi_p is None else chi_p
    chi_pp = chi if chi_pp is None else chi_pp
    if projectors is None:
        projectors = _cut_projectors(env, A, B, chi, chi_p, chi_pp, strategy, stats, renv_isos)
    C, T = env["C"], env["T"]
    site = {"a": A, "b": B}
    nC, nT = dict(C), dict(T)
    nrm = frob_normalise if normalise else (lambda t: t)
    for x in SUBS:
        y = OTHER[x]
        p_yx = projectors[y + x]
        p_xy = projectors[x + y]
        Xo = orient_left(site[x])
        if strategy == "sequential":
            nC[(y, 1)] = nrm(corner_top_left(C[(x, 1)], T[(x, 2)], p_yx["v1"], p_yx["v2"]))
            nT[(y, 1)] = nrm(absorb_truncate(T[(x, 1)], Xo, Xo, p_xy["v1"], p_xy["v2"],
                                             p_yx["v1"], p_yx["v2"]))
            nC[(x, 4)] = nrm(corner_bottom_left(C[(y, 4)], T[(y, 4)], p_yx["v1"], p_yx["v2"]))
        else:
            nC[(y, 1)] = nrm(corner_top_left_one_shot(C[(x, 1)], T[(x, 2)], p_yx["V"]))
            nT[(y, 1)] = nrm(absorb_one_shot(T[(x, 1)], Xo, Xo, p_xy["V"], p_yx["V"]))
            nC[(x, 4)] = nrm(corner_bottom_left_one_shot(C[(y, 4)], T[(y, 4)], p_yx["V"]))
    return {"C": nC, "T": nT}, projectors


def left_move(env, A, B, chi, chi_p=None, chi_pp=None, strategy="sequential", stats=None):
    """Left move = two column absorptions, projectors recomputed for the second column
    (P:L43 'That completes a full left move'; reading R4)."""
    env, _ = column_absorption(env, A, B, chi, chi_p, chi_pp, strategy, stats)
    env, _ = column_absorption(env, A, B, chi, chi_p, chi_pp, strategy, stats)
    return env


# ----------------------------------------------------------------------------------
# Rotations: moves in the other three directions (P:L43 'Moves in other directions can
# be adjusted accordingly'); clockwise storage makes a 90 deg turn a relabelling.
# ----------------------------------------------------------------------------------

def rotate_cw(env, A, B):
    """Rotate the picture 90 deg clockwise: left edge -> top edge etc.  Environment
    tensors are relabelled k -> k+1 with no data movement (clockwise storage); the site
    legs (s,u,l,d,r) become (s, l, d, r, u) i.e. A' = A.transpose(0,2,3,4,1)."""
    nC = {(x, k % 4 + 1): v for (x, k), v in env["C"].items()}
    nT = {(x, k % 4 + 1): v for (x, k), v in env["T"].items()}
    return {"C": nC, "T": nT}, A.transpose(0, 2, 3, 4, 1), B.transpose(0, 2, 3, 4, 1)


def rotate_ccw(env, A, B):
    nC = {(x, (k - 2) % 4 + 1): v for (x, k), v in env["C"].items()}
    nT = {(x, (k - 2) % 4 + 1): v for (x, k), v in env["T"].items()}
    return {"C": nC, "T": nT}, A.transpose(0, 4, 1, 2, 3), B.transpose(0, 4, 1, 2, 3)


_TURNS = {"left": 0, "down": 1, "right": 2, "up": 3}   # clockwise quarter turns bringing
                                                       # that side to the left


def move(env, A, B, direction, chi, chi_p=None, chi_pp=None, strategy="sequential", stats=None):
    """Directional move by rotate -> left move -> rotate back."""
    n = _TURNS[direction]
    e, a, b = env, A, B
    for _ in range(n):
        e, a, b = rotate_cw(e, a, b)
    e = left_move(e, a, b, chi, chi_p, chi_pp, strategy, stats)
    for _ in range(n):
        e, a, b = rotate_ccw(e, a, b)
    return e


def ctm_iteration(env, A, B, chi, chi_p=None, chi_pp=None, strategy="sequential", stats=None):
    """One CTM iteration = left, right, up, down moves (reading R17)."""
    for d in ("left", "right", "up", "down"):
        env = move(env, A, B, d, chi, chi_p, chi_pp, strategy, stats)
    return env


# ----------------------------------------------------------------------------------
# Convergence of the CTM iteration ("After applying moves in four directions
# N_CTM ~ 10-30 times, the environment tensors will become sufficiently converged";
# criterion: reading R22 -- sorted corner spectra normalised to unit 1-norm, distance =
# max over the 8 corners of the 1-norm of the difference, zero-padded)
# ----------------------------------------------------------------------------------

def corner_spectrum(C):
    """Singular values of a corner, descending, normalised to unit sum (reading R22)."""
    s = np.linalg.svd(C, compute_uv=False)
    return s / s.sum()


def corner_spectra(env):
    return {key: corner_spectrum(C) for key, C in env["C"].items()}


def spectra_distance(sp1, sp2):
    """max over corners of sum_i |s_i - s'_i| (the shorter spectrum zero-padded)."""
    out = 0.0
    for key in sp1:
        a, b = sp1[key], sp2[key]
        n = max(a.size, b.size)
        a = np.pad(a, (0, n - a.size))
        b = np.pad(b, (0, n - b.size))
        out = max(out, float(np.abs(a - b).sum()))
    return out


def converge(env, A, B, chi, tol, max_iter, chi_p=None, chi_pp=None, strategy="sequential"):
    """CTM iterations until the corner spectra move by less than tol between iterations
    (reading R22), at most max_iter.  Returns (env, iterations, last distance)."""
    prev = corner_spectra(env)
    delta = np.inf
    for it in range(1, max_iter + 1):
        env = ctm_iteration(env, A, B, chi, chi_p, chi_pp, strategy)
        cur = corner_spectra(env)
        delta = spectra_distance(prev, cur)
        if delta < tol:
            return env, it, delta
        prev = cur
    return env, max_iter, delta


# ----------------------------------------------------------------------------------
# Closures (Fig 1(c,d); observables implied by P:L92)
# ----------------------------------------------------------------------------------

def double_layer(X, Xb=None):
    """a = sum_s X X* (Fig 1(b)), legs split (uk,ub,lk,lb,dk,db,rk,rb)."""
    Xb = X if Xb is None else Xb
    return _c("sabcd,sefgh->aebfcgdh", X, Xb)


def norm_2x2(env, A, B):
    """<psi|psi> on the 2x2 patch of Fig 1(d) = Tr(E_ul E_ur E_lr E_ll); each
    enlarged corner is a corner, two edges and a double-layer site (split ket/bra legs).
        C_a^1  T_a^2  T_b^2  C_b^2
        T_a^1    A      B    T_b^3
        T_b^1    B      A    T_a^3
        C_b^4  T_b^4  T_a^4  C_a^3"""
    C, T = env["C"], env["T"]
    # E_ul: C_a^1(d=x, r=y) T_a^2(l=y, k, b, r=Y) T_a^1(d=X, l, m, u=x) A(s,k,l,d,r) A*(s,b,m,e,q)
    E = _c("xy,ykbY->xkbY", C[("a", 1)], T[("a", 2)])
    E = _c("xkbY,Xlmx->kbYXlm", E, T[("a", 1)])
    E = _c("kbYXlm,skldr->bYXmsdr", E, A)
    Eul = _c("bYXmsdr,sbmeq->YrqXde", E, A)            # (Y, kr, br, X, kd, bd)
    # E_ur: T_b^2(l=Y, k, b, r=z) C_b^2(l=z, d=w) T_b^3(u=w, l, m, d=W) B(s,k,t,d,l) B*(s,b,u,e,m)
    E = _c("Ykbz,zw->Ykbw", T[("b", 2)], C[("b", 2)])
    E = _c("Ykbw,wlmW->YkblmW", E, T[("b", 3)])
    E = _c("YkblmW,sktdl->YbmWstd", E, B)
    Eur = _c("YbmWstd,sbuem->YtuWde", E, B)            # (Y, kl, bl, W, kd, bd)
    # E_lr: T_a^3(u=W, k, b, d=v) C_a^3(u=v, l=V) T_a^4(r=V, m, n, l=U) A(s,u,t,m,k) A*(s,p,q,n,b)
    E = _c("Wkbv,vV->WkbV", T[("a", 3)], C[("a", 3)])
    E = _c("WkbV,VmnU->WkbmnU", E, T[("a", 4)])
    E = _c("WkbmnU,sutmk->WbnUsut", E, A)
    Elr = _c("WbnUsut,spqnb->WUutpq", E, A)            # (W, U, ku, kl, bu, bl)
    # E_ll: T_b^4(r=U, k, b, l=Z) C_b^4(r=Z, u=z) T_b^1(d=z, l, m, u=X) B(s,u,l,k,r) B*(s,p,m,b,q)
    E = _c("UkbZ,Zz->Ukbz", T[("b", 4)], C[("b", 4)])
    E = _c("Ukbz,zlmX->UkblmX", E, T[("b", 1)])
    E = _c("UkblmX,sulkr->UbmXsur", E, B)
    Ell = _c("UbmXsur,spmbq->UXurpq", E, B)            # (U, X, ku, kr, bu, br)
    # ring: top bond Y and A-B bond (r,q); right bond W and B-A bond (f,g);
    #       bottom bond U and A-B bond (h,i); left bond X and A-B bond (d,e)
    R = _c("YrqXde,YrqWfg->XdeWfg", Eul, Eur)
    R = _c("XdeWfg,WUfhgi->XdeUhi", R, Elr)
    return float(_c("XdeUhi,UXdhei->", R, Ell))


def bond_rho(env, A, B, bond="H"):
    """Two-site reduced density matrix rho(s_A, s_B, t_A, t_B) (ket A, ket B, bra A, bra B),
    unnormalised, on the 2x1 window (bond 'H', reading R18)
        C_a^1  T_a^2  T_b^2  C_b^2
        T_a^1    A      B    T_b^3
        C_a^4  T_a^4  T_b^4  C_b^3
    or (bond 'V') the same window after a counter-clockwise turn, which brings the
    vertical A-over-B bond {C_a^1,T_a^2,C_a^2 / T_a^1,A,T_a^3 / T_b^1,B,T_b^3 /
    C_b^4,T_b^4,C_b^3} to this horizontal form."""
    if bond == "V":
        env_r, Ar, Br = rotate_ccw(env, A, B)
        return bond_rho(env_r, Ar, Br, "H")
    if bond != "H":
        raise ValueError(bond)
    C, T = env["C"], env["T"]
    # left half: C_a^1(d=x, r=y) T_a^1(d=X, k, b, u=x) C_a^4(r=Z, u=X) T_a^2(l=y, m, n, r=Y)
    #            T_a^4(r=U, p, q, l=Z) A(s, u=m, l=k, d=p, r) A*(t, u=n, l=b, d=q, r=w)
    L = _c("xy,Xkbx->ykbX", C[("a", 1)], T[("a", 1)])
    L = _c("ykbX,ZX->ykbZ", L, C[("a", 4)])
    L = _c("ykbZ,ymnY->kbZmnY", L, T[("a", 2)])
    L = _c("kbZmnY,UpqZ->kbmnYUpq", L, T[("a", 4)])
    L = _c("kbmnYUpq,smkpr->bnYUqsr", L, A)
    L = _c("bnYUqsr,tnbqw->YUsrtw", L, A)                # (Y, U, sA, kr, tA, br)
    # right half: T_b^2(l=Y, m, n, r=z) C_b^2(l=z, d=c) T_b^3(u=c, k, l, d=W) C_b^3(u=W, l=V)
    #             T_b^4(r=V, p, q, l=U) B(S, u=m, l=r, d=p, r=k) B*(T, u=n, l=w, d=q, r=l)
    R = _c("Ymnz,zc->Ymnc", T[("b", 2)], C[("b", 2)])
    R = _c("Ymnc,cklW->YmnklW", R, T[("b", 3)])
    R = _c("YmnklW,WV->YmnklV", R, C[("b", 3)])
    R = _c("YmnklV,VpqU->YmnklUpq", R, T[("b", 4)])
    R = _c("YmnklUpq,Smrpk->YnlUqSr", R, B)
    R = _c("YnlUqSr,Tnwql->YUSrTw", R, B)               # (Y, U, sB, kl, tB, bl)
    return _c("YUsrtw,YUSrTw->sStT", L, R)


def site_spins(env, A, B):
    """Single-site spin expectations <S^x>, <S^z> (S = sigma/2, d = 2; <S^y> = 0 for the
    real states here) of A and B from the 2x1-window rho of the H bond by partial trace
    ("staggered magnetization"; reading R23).  Returns ((Sx_A, Sz_A),
    (Sx_B, Sz_B))."""
    rho = bond_rho(env, A, B, "H")                      # (sA, sB, tA, tB)
    rA = np.einsum("sutu->st", rho)
    rB = np.einsum("usut->st", rho)
    sx = np.array([[0.0, 0.5], [0.5, 0.0]])
    sz = np.array([[0.5, 0.0], [0.0, -0.5]])
    out = []
    for r in (rA, rB):
        r = 0.5 * (r + r.T) / np.trace(r)
        out.append((float(np.trace(r @ sx)), float(np.trace(r @ sz))))
    return tuple(out)


def staggered_magnetization(env, A, B):
    """m_s = (|<S>_A| + |<S>_B|) / 2 (reading R23)."""
    (xa, za), (xb, zb) = site_spins(env, A, B)
    return 0.5 * (np.hypot(xa, za) + np.hypot(xb, zb))


def rho_matrix(rho):
    """rho(sA,sB,tA,tB) -> (sA sB) x (tA tB) matrix, symmetrised (rho + rho^T)/2
     and divided by its trace."""
    dA, dB = rho.shape[0], rho.shape[1]
    m = rho.reshape(dA * dB, dA * dB)
    m = 0.5 * (m + m.T)
    return m / np.trace(m)


def bond_energy(env, A, B, h, bond="H"):
    """e = Tr(rho h) / Tr rho for the bond operator h(s_i,s_j,s_i',s_j') = <s_i s_j|h|s_i' s_j'>
    (PAPER Eq. (1); reading R14: h = S.S, S = sigma/2).  Returns (e, rho matrix)."""
    m = rho_matrix(bond_rho(env, A, B, bond))
    H = h.reshape(m.shape)
    return float(np.trace(m @ H)), m

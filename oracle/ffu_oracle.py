"""CPU float64 oracle for the imaginary-time evolution step of arXiv 2306.08212 (SURVEY.md
8(f) item 4): second-order Suzuki-Trotter gates applied bond by bond with the fast full
update (FFU) against the CTM environment.

TEST INFRASTRUCTURE ONLY (same rules as oracle/ctm_oracle.py): only tests/, smoke() and
bench.py's reference/cpu_baseline legs may import it; it shares no code with the CUDA path.

The paper states the method in one passage (Results): "We used imaginary-time
evolution method with a second-order Suzuki-Trotter decomposition to optimize iPEPS tensors
for ground state ... we applied the fast full update scheme (FFU) as described in Ref
[iPEPS1] to avoid recomputing the effective environments after each update step ... start
optimization with a large imaginary time delta ~ 0.1 ... decrease delta until it reaches
delta ~ 1e-4 ... we also implemented the gauge-fixing step".  Everything it leaves to the
cited reference is fixed by the readings R25-R30 of DESIGN.md, restated where used:

  R25  gate g(delta) = exp(-delta h) on one bond, h (d,d,d,d) as (s_i, s_j, s_i', s_j'),
       by the eigendecomposition of the d^2 x d^2 matrix (exact exponential).
  R26  bond reduction: A (s,u,l,d,r) = X (u,l,d,w) aR (w,s,r) with X the left singular
       vectors of A as (u l d) x (s r) (sign rule of SURVEY 0) and aR = X^T A; B = bL (s,l,v)
       Y (v,u,d,r) likewise from B as (u d r) x (s l).  (The cited full update uses a QR;
       the SVD fixes the gauge of w so the GPU and the oracle agree entrywise.)
  R27  bond environment N(w, v; w', v') = the 2x1 window of reading R18 with A, B replaced
       by X, Y (their physical and bond legs left open through w, v), made symmetric and
       positive: eigenvalues clipped at 0, plus 1e-12 max|lambda| (SPEC's positivisation).
  R28  split: theta'(w,s,t,v) = sum g(s,t,s',t') aR(w,s',r) bL(t',r,v) ... truncated back to
       bond D by alternating least squares in the N metric, started from the truncated SVD of
       theta' (sign rule; aR = U sqrt(S), bL = sqrt(S) V^T), a fixed number of sweeps (each:
       solve for aR with bL fixed, then for bL with aR fixed), the normal matrices regularised
       by 1e-12 tr/n.  The gauge-fixing step of the cited reference is a conditioning aid that
       leaves the optimum unchanged; it is not applied.
  R29  second-order Trotter step over the four bonds of the 2-site unit cell, H1 = A left of
       B, H2 = B left of A, V1 = A above B, V2 = B above A (Strang splitting):
       H1(d/2) H2(d/2) V1(d/2) V2(d) V1(d/2) H2(d/2) H1(d/2).
  R30  FFU: after every bond update the environment is refreshed by ONE CTM iteration (left,
       right, up, down moves) instead of being reconverged.
"""
from __future__ import annotations

import numpy as np

from . import ctm_oracle as O


def _c(spec, x, y):
    return np.einsum(spec, x, y, optimize=True)


# ------------------------------------------------------------------------------------
# R25 gate
# ------------------------------------------------------------------------------------
def trotter_gate(h: np.ndarray, delta: float) -> np.ndarray:
    """g = exp(-delta h) ("imaginary-time evolution"), h (d,d,d,d) -> g (d,d,d,d)."""
    d = h.shape[0]
    H = h.reshape(d * d, d * d)
    H = 0.5 * (H + H.T)
    w, V = np.linalg.eigh(H)
    return ((V * np.exp(-delta * w)) @ V.T).reshape(d, d, d, d)


# ------------------------------------------------------------------------------------
# R26 bond reduction (horizontal bond: A's r leg = B's l leg)
# ------------------------------------------------------------------------------------
def reduce_left(A):
    """A (s,u,l,d,r) = X (u,l,d,w) aR (w,s,r): X = left singular vectors (sign rule) of
    A as (u l d) x (s r), m = min(D^3, d D) columns; aR = X^T A."""
    d, D = A.shape[0], A.shape[1]
    Am = A.transpose(1, 2, 3, 0, 4).reshape(D ** 3, d * D)
    m = min(D ** 3, d * D)
    X = O.left_singular(Am, m)
    aR = (X.T @ Am).reshape(m, d, D)
    return X.reshape(D, D, D, m), aR


def reduce_right(B):
    """B (s,u,l,d,r) = bL (s,l,v) Y (v,u,d,r): Y^T = left singular vectors (sign rule) of
    B as (u d r) x (s l); bL = B Y^T."""
    d, D = B.shape[0], B.shape[1]
    Bm = B.transpose(1, 3, 4, 0, 2).reshape(D ** 3, d * D)     # (u d r) x (s l)
    m = min(D ** 3, d * D)
    Yt = O.left_singular(Bm, m)                                  # (u d r) x v
    bL = (Yt.T @ Bm).reshape(m, d, D).transpose(1, 2, 0)        # (s, l, v)
    return bL, Yt.T.reshape(m, D, D, D)                          # Y (v, u, d, r)


# ------------------------------------------------------------------------------------
# R27 bond environment (2x1 window of reading R18 with X, Y in place of A, B)
# ------------------------------------------------------------------------------------
def bond_env_h(env, X, Y):
    """N(w, v, w', v'): the 2x1 window
        C_a^1  T_a^2  T_b^2  C_b^2
        T_a^1    X      Y    T_b^3
        C_a^4  T_a^4  T_b^4  C_b^3
    with ket X, Y and bra X*, Y*, their open legs w, v (ket) and w', v' (bra)."""
    C, T = env["C"], env["T"]
    # left half (as ctm_oracle.bond_rho): X (u=m, l=k, d=p, w) / X* (u=n, l=b, d=q, w')
    L = _c("xy,Xkbx->ykbX", C[("a", 1)], T[("a", 1)])
    L = _c("ykbX,ZX->ykbZ", L, C[("a", 4)])
    L = _c("ykbZ,ymnY->kbZmnY", L, T[("a", 2)])
    L = _c("kbZmnY,UpqZ->kbmnYUpq", L, T[("a", 4)])
    L = _c("kbmnYUpq,mkpw->bnYUqw", L, X)
    L = _c("bnYUqw,nbqe->YUwe", L, X)                            # (Y, U, w, w')
    # right half: Y (v, u=m, d=p, r=k) / Y* (v', u=n, d=q, r=l)
    R = _c("Ymnz,zc->Ymnc", T[("b", 2)], C[("b", 2)])
    R = _c("Ymnc,cklW->YmnklW", R, T[("b", 3)])
    R = _c("YmnklW,WV->YmnklV", R, C[("b", 3)])
    R = _c("YmnklV,VpqU->YmnklUpq", R, T[("b", 4)])
    R = _c("YmnklUpq,fmpk->YnlUqf", R, Y)
    R = _c("YnlUqf,gnql->YUfg", R, Y)                            # (Y, U, v, v')
    return _c("YUwe,YUfg->wfeg", L, R)                          # (w, v, w', v')


def positivise(N):
    """Symmetrise N as (w v) x (w' v') and clip its spectrum at 0 (+ 1e-12 max|lambda|)."""
    m1, m2 = N.shape[0], N.shape[1]
    M = N.reshape(m1 * m2, m1 * m2)
    M = 0.5 * (M + M.T)
    lam, V = np.linalg.eigh(M)
    lam = np.maximum(lam, 0.0) + 1e-12 * np.abs(lam).max()
    return ((V * lam) @ V.T).reshape(m1, m2, m1, m2)


# ------------------------------------------------------------------------------------
# R28 gate + ALS split
# ------------------------------------------------------------------------------------
def apply_gate(aR, bL, g):
    """theta'(w, s, t, v) = sum g(s,t,s',t') aR(w,s',r) bL(t',r,v)."""
    th = _c("wsr,trv->wstv", aR, bL)
    return _c("stpq,wpqv->wstv", g, th)


def svd_split(theta, D):
    """Truncated SVD of theta as (w s) x (t v) keeping D (sign rule): aR = U sqrt(S),
    bL(t, r, v) = (sqrt(S) V^T)."""
    m1, d1, d2, m2 = theta.shape
    Mt = theta.reshape(m1 * d1, d2 * m2)
    n = min(D, m1 * d1, d2 * m2)
    U = O.left_singular(Mt, n)                       # (w s) x n
    SVt = U.T @ Mt                                   # n x (t v) = S V^T
    s = np.sqrt(np.maximum(np.linalg.norm(SVt, axis=1), 1e-300))
    aR = (U * s).reshape(m1, d1, n)
    bL = (SVt / s[:, None]).reshape(n, d2, m2).transpose(1, 0, 2)   # (t, r, v)
    return aR, bL


def _regularised_solve(Q, b):
    n = Q.shape[0]
    Q = 0.5 * (Q + Q.T) + 1e-12 * np.trace(Q) / n * np.eye(n)
    return np.linalg.solve(Q, b)


def als_split(theta, N, D, sweeps):
    """Minimise ||aR bL - theta||_N over bond-D pairs (R28), `sweeps` alternations from the
    truncated SVD.  Returns (aR, bL, [cost after each half-step])."""
    aR, bL = svd_split(theta, D)
    m1, d1, d2, m2 = theta.shape
    n = aR.shape[2]
    Nt = _c("wvxy,xsty->wstv", N, theta)              # N theta' (ket side open)
    tNt = float(np.einsum("wstv,wstv->", theta, Nt))
    costs = []
    for _ in range(sweeps):
        # aR with bL fixed: Q_a[(w,r),(w',r')] = sum_{t,v,v'} bL(t,r,v) N(w,v,w',v') bL(t,r',v')
        Qa = np.einsum("trv,wvxy,tsy->wrxs", bL, N, bL).reshape(m1 * n, m1 * n)
        ba = np.einsum("trv,wstv->wrs", bL, Nt).reshape(m1 * n, d1)
        aR = _regularised_solve(Qa, ba).reshape(m1, n, d1).transpose(0, 2, 1)
        # bL with aR fixed: Q_b[(r,v),(r',v')] = sum_{s,w,w'} aR(w,s,r) N(w,v,w',v') aR(w',s,r')
        Qb = np.einsum("wsr,wvxy,xsq->rvqy", aR, N, aR).reshape(n * m2, n * m2)
        bb = np.einsum("wsr,wstv->rvt", aR, Nt).reshape(n * m2, d2)
        bL = _regularised_solve(Qb, bb).reshape(n, m2, d2).transpose(2, 0, 1)
        phi = _c("wsr,trv->wstv", aR, bL)
        costs.append(float(np.einsum("wstv,wvxy,xsty->", phi, N, phi)
                           - 2 * np.einsum("wstv,wstv->", phi, Nt) + tNt))
    return aR, bL, costs


# ------------------------------------------------------------------------------------
# one bond update (horizontal, A left of B) and the Trotter step
# ------------------------------------------------------------------------------------
def bond_update_h(env, A, B, g, D, sweeps):
    """FFU update of the horizontal bond A (left) - B (right) (R26-R28).  Returns the new
    (A', B'), each Frobenius-normalised, and the ALS costs."""
    X, aR = reduce_left(A)
    bL, Y = reduce_right(B)
    N = positivise(bond_env_h(env, X, Y))
    th = apply_gate(aR, bL, g)
    aR2, bL2, costs = als_split(th, N, D, sweeps)
    A2 = _c("uldw,wsr->suldr", X, aR2)
    B2 = _c("slv,vudr->suldr", bL2, Y)
    return A2 / np.linalg.norm(A2), B2 / np.linalg.norm(B2), costs


def swap_sublattices(env):
    """Relabel a <-> b (the window with B on the left of A is the A-left window with the
    sublattice labels exchanged: the environment tensors are labelled by their adjacent site,
    reading R2)."""
    sw = {"a": "b", "b": "a"}
    return {"C": {(sw[x], k): v for (x, k), v in env["C"].items()},
            "T": {(sw[x], k): v for (x, k), v in env["T"].items()}}


def bond_update(env, A, B, g, D, sweeps, bond):
    """bond in H1 (A left of B), H2 (B left of A), V1 (A above B), V2 (B above A).
    Vertical bonds: the picture is turned counter-clockwise (ctm_oracle.rotate_ccw) so the
    upper site is on the left, updated as H, and the sites are turned back."""
    if bond == "H1":
        return bond_update_h(env, A, B, g, D, sweeps)
    if bond == "H2":
        B2, A2, c = bond_update_h(swap_sublattices(env), B, A, g, D, sweeps)
        return A2, B2, c
    e, a, b = O.rotate_ccw(env, A, B)
    if bond == "V1":
        a2, b2, c = bond_update_h(e, a, b, g, D, sweeps)
    elif bond == "V2":
        b2, a2, c = bond_update_h(swap_sublattices(e), b, a, g, D, sweeps)
    else:
        raise ValueError(bond)
    # turn the sites back (one clockwise quarter turn: (s,u,l,d,r) -> (s,l,d,r,u) inverse)
    _, A2, B2 = O.rotate_cw({"C": {}, "T": {}}, a2, b2)
    return A2, B2, c


TROTTER_ORDER = (("H1", 0.5), ("H2", 0.5), ("V1", 0.5), ("V2", 1.0), ("V1", 0.5), ("H2", 0.5), ("H1", 0.5))


def trotter_step(env, A, B, h, delta, D, chi, sweeps, refresh=True):
    """One second-order Trotter step (R29) with the FFU environment refresh (R30).
    Returns (env, A, B, [ALS costs per bond])."""
    log = []
    gates = {f: trotter_gate(h, f * delta) for f in (0.5, 1.0)}
    for bond, f in TROTTER_ORDER:
        A, B, costs = bond_update(env, A, B, gates[f], D, sweeps, bond)
        log.append(costs)
        if refresh:
            env = O.ctm_iteration(env, A, B, chi)
    return env, A, B, log

"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method: it only draws the input tensors of
SURVEY.md 8(d) ("Synthetic inputs") so that `oracle/` and `paper_2306_08212_b200/`
see bit-identical arrays.  Neither side imports the other; both import this.

Paper workloads (Sec. V): Heisenberg ground states, d = 2, D = 2..14,
chi ~ 10(D+1).  The optimised iPEPS tensors are not published, so seeded Gaussian
tensors stand in for them:

  * A, B (d,D,D,D,D) as (s,u,l,d,r): i.i.d. N(0,1); for the "decaying" configs each
    virtual leg is scaled by s_k = exp(-k/2), k = 0..D-1 (BASELINE.json configs 3-5);
    then divided by the Frobenius norm.
  * C (chi,chi): N(0,1) / ||.||_F.
  * T (chi,D,D,chi): N(0,1), symmetrised across the ket/bra pair
    T <- (T + T.swapaxes(1,2))/2, then / ||.||_F.

Storage order ("clockwise"):  every boundary tensor is stored walking
the boundary clockwise, T^1 (d,k,b,u), T^2 (l,k,b,r), T^3 (u,k,b,d), T^4 (r,k,b,l),
C^1 (d,r), C^2 (l,d), C^3 (u,l), C^4 (r,u).  k/b are the ket/bra legs facing the bulk.

Generator: numpy Generator(PCG64(seed)), standard_normal, float64, drawn in the order
A, B, C_x^k (x in a,b; k = 1..4), T_x^k (x in a,b; k = 1..4).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 230608212

SUBS = ("a", "b")
DIRS = (1, 2, 3, 4)


@dataclass(frozen=True)
class Config:
    name: str
    index: int          # seed offset (seed = 230608212 + config index)
    d: int
    D: int
    chi: int            # target boundary dimension chi
    chi_p: int          # chi'  (first sequential isometry)
    chi_pp: int         # chi'' (appendix side isometries)
    decaying: bool      # decaying virtual spectrum s_k = exp(-k/2)
    chi0: int | None = None   # initial boundary extent (None -> chi)
    iterations: int = 20
    notes: str = field(default="", compare=False)

    @property
    def seed(self) -> int:
        return SEED_BASE + self.index

    @property
    def chi_init(self) -> int:
        return self.chi if self.chi0 is None else self.chi0


# BASELINE.json "configs" (index 0..4).  chi = chi' = chi'' (PAPER L90 reading,
# DESIGN.md reading R9).
CONFIGS = {
    "tiny": Config("tiny", 0, 2, 2, 8, 8, 8, False, iterations=1),
    "c2": Config("c2", 1, 2, 4, 32, 32, 32, False),
    "c3": Config("c3", 2, 2, 6, 64, 64, 64, True),
    "c4": Config("c4", 3, 2, 8, 128, 128, 128, True),
    "c5": Config("c5", 4, 2, 10, 200, 200, 200, True),
    "c5_256": Config("c5_256", 4, 2, 10, 256, 256, 256, True),
    # converging variants (reading R16b): partial-trace start, chi = D^2 so every boundary
    # extent equals chi from the first move; used for the 1e-9 gauge-invariant parity.
    "c2_dl": Config("c2_dl", 1, 2, 4, 16, 16, 16, False),
    "c3_dl": Config("c3_dl", 2, 2, 6, 36, 36, 36, True),
    "c4_dl": Config("c4_dl", 3, 2, 8, 64, 64, 64, True),
}
ENV_INIT = {"c2_dl": "double_layer", "c3_dl": "double_layer", "c4_dl": "double_layer"}


def custom(d: int, D: int, chi: int, *, chi_p: int | None = None, chi_pp: int | None = None,
           chi0: int | None = None, decaying: bool = False, seed_index: int = 0,
           name: str = "custom") -> Config:
    return Config(name, seed_index, d, D, chi, chi if chi_p is None else chi_p,
                  chi if chi_pp is None else chi_pp, decaying, chi0)


def _site(rng: np.random.Generator, d: int, D: int, decaying: bool) -> np.ndarray:
    A = rng.standard_normal((d, D, D, D, D))
    if decaying:
        s = np.exp(-np.arange(D) / 2.0)
        A = A * s[None, :, None, None, None] * s[None, None, :, None, None] \
              * s[None, None, None, :, None] * s[None, None, None, None, :]
    return A / np.linalg.norm(A)


def generate(cfg: Config, env_init: str | None = None) -> dict:
    """Return {'A','B', 'C': {(x,k): arr}, 'T': {(x,k): arr}} in clockwise storage.

    env_init "gaussian" is BASELINE.json's recipe.  "double_layer" (DESIGN.md reading
    R16b) replaces the boundary tensors by the standard partial-trace start of CTM
    (trace the outward legs of the double-layer site), a positive
    environment for which CTM converges smoothly; the same seeded A, B are used."""
    if env_init is None:
        env_init = ENV_INIT.get(cfg.name, "gaussian")
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    A = _site(rng, cfg.d, cfg.D, cfg.decaying)
    B = _site(rng, cfg.d, cfg.D, cfg.decaying)
    c0 = cfg.chi_init
    C, T = {}, {}
    for x in SUBS:
        for k in DIRS:
            c = rng.standard_normal((c0, c0))
            C[(x, k)] = c / np.linalg.norm(c)
    for x in SUBS:
        for k in DIRS:
            t = rng.standard_normal((c0, cfg.D, cfg.D, c0))
            t = 0.5 * (t + t.swapaxes(1, 2))
            T[(x, k)] = t / np.linalg.norm(t)
    if env_init == "double_layer":
        C, T = _partial_trace_env(A, B)
    elif env_init != "gaussian":
        raise ValueError(env_init)
    return {"A": A, "B": B, "C": C, "T": T}


def _partial_trace_env(A, B):
    """Boundary from the double-layer sites with the outward legs traced (ket = bra),
    boundary extent D^2 (grows to chi over the first moves).  Input preparation only:
    the fused legs keep the clockwise storage order of the module docstring."""
    D = A.shape[1]
    D2 = D * D
    site = {"a": A, "b": B}
    C, T = {}, {}
    for x, y in (("a", "b"), ("b", "a")):
        ax = np.einsum("sabcd,sefgh->aebfcgdh", site[x], site[x])   # (uk,ub,lk,lb,dk,db,rk,rb)
        ay = np.einsum("sabcd,sefgh->aebfcgdh", site[y], site[y])
        # corners: the diagonal neighbour has x's sublattice; edges: the neighbour is y
        C[(x, 1)] = np.einsum("aabbcdef->cdef", ax).reshape(D2, D2)          # (d, r)
        C[(x, 2)] = np.einsum("aacdefbb->cdef", ax).reshape(D2, D2)          # (l, d)
        C[(x, 3)] = np.einsum("cdefaabb->cdef", ax).reshape(D2, D2)          # (u, l)
        C[(x, 4)] = np.einsum("cdaabbef->efcd", ax).reshape(D2, D2)          # (r, u)
        T[(x, 1)] = np.einsum("uvaadekb->dekbuv", ay).reshape(D2, D, D, D2)  # (d, k, b, u)
        T[(x, 2)] = np.einsum("aalmkbrs->lmkbrs", ay).reshape(D2, D, D, D2)  # (l, k, b, r)
        T[(x, 3)] = np.einsum("uvkbdeaa->uvkbde", ay).reshape(D2, D, D, D2)  # (u, k, b, d)
        T[(x, 4)] = np.einsum("kblmaars->rskblm", ay).reshape(D2, D, D, D2)  # (r, k, b, l)
    C = {k: v / np.linalg.norm(v) for k, v in C.items()}
    T = {k: v / np.linalg.norm(v) for k, v in T.items()}
    return C, T


def random_isometries(rng: np.random.Generator, chi: int, D: int, chi_p: int, chi_out: int):
    """Random (v1, v2) pair with v1 (chi,D,chi') and v2 (chi',D,chi_out), columns orthonormal.

    Used only to feed *identical* isometries to both sides of the absorb/corner parity
    tests (SURVEY 8(c) "identical isometries").  QR of a Gaussian is input drawing, not
    the method's arithmetic."""
    g1 = rng.standard_normal((chi * D, chi_p))
    q1, _ = np.linalg.qr(g1)
    g2 = rng.standard_normal((chi_p * D, chi_out))
    q2, _ = np.linalg.qr(g2)
    return q1.reshape(chi, D, chi_p), q2.reshape(chi_p, D, chi_out)


def heisenberg_h() -> np.ndarray:
    """h = S.S with S = sigma/2 (PAPER Eq. (1), sign reading R14), shape (d,d,d,d) as
    (s_i, s_j, s_i', s_j'), basis |0> = up.  Written out from the Pauli matrices."""
    sx = np.array([[0, 1], [1, 0]], dtype=complex) / 2
    sy = np.array([[0, -1j], [1j, 0]], dtype=complex) / 2
    sz = np.array([[1, 0], [0, -1]], dtype=complex) / 2
    h = np.kron(sx, sx) + np.kron(sy, sy) + np.kron(sz, sz)
    assert np.allclose(h.imag, 0)
    return np.ascontiguousarray(h.real.reshape(2, 2, 2, 2))

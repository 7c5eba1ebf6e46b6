"""GPU parity: libctm (through the C ABI) against the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north star):
  * given identical isometries, contraction outputs agree entrywise within 1e-11 relative
    max-norm (fp64);
  * the gauge-free reduced environment M within 1e-10;
  * gauge-invariant quantities (2x2 norm, rho, bond energy) after fixed iterations within
    1e-9 relative.
"""
import numpy as np
import pytest

import ctm_inputs as ci
from oracle import ctm_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2306_08212_b200 import ctm
DEV = "cuda"
SVDS = ["gesvdp", "gram", "iso"]


def svd_algo(name):
    return {"gesvdp": ctm.CTM_SVD_GESVDP, "gram": ctm.CTM_SVD_GRAM, "iso": ctm.CTM_SVD_ISO}[name]


def rel_err(got, ref):
    return np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-300)


def T_(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def _iso_from_flat(p, chi, D, chi_p):
    n1, n2 = chi * D * chi_p, chi_p * D * chi
    out, off = [], 0
    for a in range(2):
        proj = {}
        for cut in ("ab", "ba"):
            proj[cut] = {"v1": p[off:off + n1].reshape(chi, D, chi_p),
                         "v2": p[off + n1:off + n1 + n2].reshape(chi_p, D, chi)}
            off += n1 + n2
        out.append(proj)
    return out


# ----------------------------------------------------------------------------------------
# rows a6-a8: absorb/truncate chain with identical isometries
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("d,D,chi,chi_p", [(2, 2, 8, 8), (2, 4, 32, 32), (2, 3, 37, 29), (2, 6, 64, 64),
                                           (2, 8, 128, 128), (2, 10, 200, 200), (2, 10, 256, 256)])
def test_absorb_truncate_identical_isometries(d, D, chi, chi_p):
    rng = np.random.default_rng(1000 + chi)
    T = rng.standard_normal((chi, D, D, chi))
    X = rng.standard_normal((d, D, D, D, D))      # (s, in, face, out, far)
    Xb = rng.standard_normal((d, D, D, D, D))     # bra != ket: catches ket/bra mix-ups
    v1i, v2i = ci.random_isometries(rng, chi, D, chi_p, chi)
    v1o, v2o = ci.random_isometries(rng, chi, D, chi_p, chi)
    ref = O.absorb_truncate(T, X, Xb, v1i, v2i, v1o, v2o)
    h = ctm.CtmHandle(d, D, chi, chi_p, chi, flags=ctm.CTM_FLAG_MOVE_ONLY)
    out = torch.empty((chi, D, D, chi), dtype=torch.float64, device=DEV)
    h.ctm_absorb_truncate(T_(T), T_(X), T_(Xb), T_(v1i), T_(v2i), T_(v1o), T_(v2o), out)
    assert rel_err(out.cpu().numpy(), ref) <= 1e-11


# ----------------------------------------------------------------------------------------
# rows a1-a4: reduced environment (gauge-free M)
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("d,D,chi,chi_pp", [(2, 2, 8, 8), (2, 2, 4, 16), (2, 4, 32, 32), (2, 3, 20, 17),
                                            (2, 8, 128, 128)])
@pytest.mark.parametrize("svd", SVDS)
def test_reduced_env(d, D, chi, chi_pp, svd):
    cfg = ci.custom(d, D, chi, chi_pp=chi_pp, seed_index=200 + chi, decaying=D >= 6)
    g = ci.generate(cfg)
    C, T, A = g["C"], g["T"], g["A"]
    x = "a"
    M_ref, _ = O.reduced_env_approx(C[(x, 1)], T[(x, 2)], C[(x, 2)], T[(x, 1)], A, A, T[(x, 3)], chi_pp)
    h = ctm.CtmHandle(d, D, chi, chi, chi_pp, svd_algo=svd_algo(svd), flags=ctm.CTM_FLAG_MOVE_ONLY)
    M = torch.empty((chi, D, D, chi), dtype=torch.float64, device=DEV)
    h.ctm_reduced_env(T_(C[(x, 1)]), T_(T[(x, 2)]), T_(C[(x, 2)]), T_(T[(x, 1)]), T_(A), T_(A), T_(T[(x, 3)]), M)
    assert rel_err(M.cpu().numpy(), M_ref) <= 1e-10


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
@pytest.mark.parametrize("svd", SVDS)
def test_side_isometry_projectors(name, svd):
    """Row a2: the side isometries TS(C^1 T^1) and TS(C^2 T^3) span the oracle's subspaces.
    The composite V = v1 v2 is compared through its projector applied to random
    probes, P x = V (V^T x) (gauge-free), and v1 v1^T likewise."""
    cfg = ci.CONFIGS[name]
    g = ci.generate(cfg)
    C, T, A = g["C"], g["T"], g["A"]
    d, D, chi = cfg.d, cfg.D, cfg.chi
    x = "a"
    _, ref = O.reduced_env_approx(C[(x, 1)], T[(x, 2)], C[(x, 2)], T[(x, 1)], A, A, T[(x, 3)], chi)
    h = ctm.CtmHandle(d, D, chi, chi, chi, svd_algo=svd_algo(svd), flags=ctm.CTM_FLAG_MOVE_ONLY)
    M = torch.empty((chi, D, D, chi), dtype=torch.float64, device=DEV)
    n1 = min(chi, chi * D)
    n2 = min(chi, n1 * D)
    iso = torch.zeros(2 * (chi * D * n1 + n1 * D * n2), dtype=torch.float64, device=DEV)
    h.ctm_reduced_env(T_(C[(x, 1)]), T_(T[(x, 2)]), T_(C[(x, 2)]), T_(T[(x, 1)]), T_(A), T_(A), T_(T[(x, 3)]), M,
                      iso_out=iso)
    p = iso.cpu().numpy()
    off, got = 0, []
    for _ in range(2):
        v1 = p[off:off + chi * D * n1].reshape(chi, D, n1)
        off += chi * D * n1
        v2 = p[off:off + n1 * D * n2].reshape(n1, D, n2)
        off += n1 * D * n2
        got += [v1, v2]
    rng = np.random.default_rng(7)
    for side in range(2):
        v1g, v2g = got[2 * side], got[2 * side + 1]
        v1r, v2r = ref[2 * side], ref[2 * side + 1]
        a = v1g.reshape(-1, n1)
        b = v1r.reshape(-1, n1)
        X = rng.standard_normal((a.shape[0], 8))
        assert np.abs(a @ (a.T @ X) - b @ (b.T @ X)).max() <= 1e-9 * np.abs(X).max()
        Vg = np.einsum("pka,abz->pkbz", v1g, v2g).reshape(-1, n2)
        Vr = np.einsum("pka,abz->pkbz", v1r, v2r).reshape(-1, n2)
        X = rng.standard_normal((Vg.shape[0], 8))
        assert np.abs(Vg @ (Vg.T @ X) - Vr @ (Vr.T @ X)).max() <= 1e-9 * np.abs(X).max()
        assert np.allclose(a.T @ a, np.eye(n1), atol=1e-12)


def test_reduced_env_untruncated_equals_exact():
    cfg = ci.custom(2, 2, 4, chi_pp=16, seed_index=211)
    g = ci.generate(cfg)
    C, T, A = g["C"], g["T"], g["A"]
    M_ex = O.reduced_env_exact(C[("b", 1)], T[("b", 2)], C[("b", 2)], T[("b", 1)], A, A, T[("b", 3)])
    h = ctm.CtmHandle(2, 2, 4, 4, 16, flags=ctm.CTM_FLAG_MOVE_ONLY)
    M = torch.empty((4, 2, 2, 4), dtype=torch.float64, device=DEV)
    h.ctm_reduced_env(T_(C[("b", 1)]), T_(T[("b", 2)]), T_(C[("b", 2)]), T_(T[("b", 1)]), T_(A), T_(A),
                      T_(T[("b", 3)]), M)
    assert rel_err(M.cpu().numpy(), M_ex) <= 1e-10


# ----------------------------------------------------------------------------------------
# rows a1-a11: left move; GPU isometries injected into the oracle -> entrywise parity
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("name,svd", [(n, s) for n in ["tiny", "c2", "c3", "c4"] for s in SVDS]
                         + [("c5", "iso"), ("c5_256", "iso")])
def test_left_move_entrywise_with_gpu_isometries(name, svd):
    cfg = ci.CONFIGS[name]
    g = ci.generate(cfg)
    h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp, svd_algo=svd_algo(svd),
                      flags=ctm.CTM_FLAG_CHECK_FINITE | ctm.CTM_FLAG_MOVE_ONLY)
    env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
    iso = torch.zeros(h.iso_numel(), dtype=torch.float64, device=DEV)
    st = h.ctm_left_move(T_(g["A"]), T_(g["B"]), env, iso_out=iso)
    # 12 per absorption, minus the right-side TS (2 x 2 SVDs) reused by the second one
    assert st["n_svd"] == 2 * 12 - 4 and np.isfinite(st["ms_total"])
    if svd == "iso":   # every truncation (C5's l = 232 included) certified by libctm's solver
        assert st["n_svd_fallback"] == 0
    got = env.to_host()
    projs = _iso_from_flat(iso.cpu().numpy(), cfg.chi, cfg.D, cfg.chi_p)
    e = {"C": g["C"], "T": g["T"]}
    for a in range(2):
        e, _ = O.column_absorption(e, g["A"], g["B"], cfg.chi, projectors=projs[a])
    for kind in ("C", "T"):
        for key, ref in e[kind].items():
            assert rel_err(got[kind][key], ref) <= 1e-11, (kind, key)
    # the isometries themselves are isometries
    for proj in projs:
        for cut in proj.values():
            v1 = cut["v1"].reshape(-1, cfg.chi_p)
            v2 = cut["v2"].reshape(-1, cfg.chi)
            assert np.allclose(v1.T @ v1, np.eye(cfg.chi_p), atol=1e-12)
            assert np.allclose(v2.T @ v2, np.eye(cfg.chi), atol=1e-12)


def test_injected_isometries_reproduce_the_move():
    """INJECT_ISO: replaying the move with its own isometries gives the same env."""
    cfg = ci.CONFIGS["c2"]
    g = ci.generate(cfg)
    h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, flags=ctm.CTM_FLAG_MOVE_ONLY)
    iso = torch.zeros(h.iso_numel(), dtype=torch.float64, device=DEV)
    e1 = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
    h.ctm_left_move(T_(g["A"]), T_(g["B"]), e1, iso_out=iso)
    e2 = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
    st = h.ctm_left_move(T_(g["A"]), T_(g["B"]), e2, iso_in=iso)
    assert st["n_svd"] == 0
    a, b = e1.to_host(), e2.to_host()
    for kind in ("C", "T"):
        for key in a[kind]:
            assert np.array_equal(a[kind][key], b[kind][key])


# ----------------------------------------------------------------------------------------
# no truncation: the full left move is exact (gauge-invariant column contraction)
# ----------------------------------------------------------------------------------------
def test_full_move_without_truncation_matches_oracle():
    cfg = ci.custom(2, 2, 16, chi0=1, seed_index=21)
    g = ci.generate(cfg)
    h = ctm.CtmHandle(2, 2, 16, flags=ctm.CTM_FLAG_MOVE_ONLY)
    env = ctm.Env.from_host(g["C"], g["T"], 2, 16)
    h.ctm_left_move(T_(g["A"]), T_(g["B"]), env)
    got = env.to_host()
    ref = O.left_move({"C": g["C"], "T": g["T"]}, g["A"], g["B"], 16)
    for x in ("a", "b"):
        y = O.OTHER[x]
        def col(e):
            c = np.einsum("xR,yklx,zmny,Sz->RklmnS", e["C"][(x, 1)], e["T"][(x, 1)], e["T"][(y, 1)], e["C"][(y, 4)])
            return c / np.linalg.norm(c)
        assert got["T"][(x, 1)].shape == ref["T"][(x, 1)].shape == (16, 2, 2, 16)
        assert np.allclose(col(got), col(ref), atol=1e-12)


@pytest.mark.parametrize("direction", ["left", "right", "up", "down"])
def test_directional_move_gauge_invariant(direction):
    cfg = ci.custom(2, 2, 16, chi0=1, seed_index=25)
    g = ci.generate(cfg)
    h = ctm.CtmHandle(2, 2, 16, flags=ctm.CTM_FLAG_MOVE_ONLY)
    env = ctm.Env.from_host(g["C"], g["T"], 2, 16)
    h.ctm_move(direction, T_(g["A"]), T_(g["B"]), env)
    ref = O.move({"C": g["C"], "T": g["T"]}, g["A"], g["B"], direction, 16)
    n_gpu = O.norm_2x2(env.to_host(), g["A"], g["B"])
    n_ref = O.norm_2x2(ref, g["A"], g["B"])
    assert abs(n_gpu - n_ref) <= 1e-10 * abs(n_ref)


# ----------------------------------------------------------------------------------------
# closures
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["tiny", "c2"])
def test_norm_2x2(name):
    cfg = ci.CONFIGS[name]
    g = ci.generate(cfg)
    h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi)
    env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
    v, ratio = h.ctm_norm_2x2(T_(g["A"]), T_(g["B"]), env)
    ref = O.norm_2x2({"C": g["C"], "T": g["T"]}, g["A"], g["B"])
    assert abs(v - ref) <= 1e-11 * abs(ref) / max(abs(ratio), 1e-6)


def _iterate_both(name, n_iter, perturb=None, svd="gesvdp"):
    """GPU n_iter CTM iterations and the oracle's; optionally a second oracle run from an
    environment perturbed by `perturb` (relative, C tensors) to measure the problem's own
    sensitivity to rounding."""
    cfg = ci.CONFIGS[name]
    g = ci.generate(cfg)
    A, B = g["A"], g["B"]
    h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, cfg.chi_p, cfg.chi_pp, svd_algo=svd_algo(svd))
    env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
    h.ctm_iterate(T_(A), T_(B), env, n_iter)
    e = {"C": g["C"], "T": g["T"]}
    for _ in range(n_iter):
        e = O.ctm_iteration(e, A, B, cfg.chi, cfg.chi_p, cfg.chi_pp)
    e2 = None
    if perturb:
        rng = np.random.default_rng(1)
        e2 = {"C": {k: v * (1 + perturb * rng.standard_normal(v.shape)) for k, v in g["C"].items()},
              "T": dict(g["T"])}
        for _ in range(n_iter):
            e2 = O.ctm_iteration(e2, A, B, cfg.chi, cfg.chi_p, cfg.chi_pp)
    hop = ci.heisenberg_h()
    out = {"norm_gpu": h.ctm_norm_2x2(T_(A), T_(B), env)[0], "norm_ref": O.norm_2x2(e, A, B),
           "eH_gpu": h.ctm_bond_energy(T_(A), T_(B), env, T_(hop), ctm.CTM_BOND_H),
           "eV_gpu": h.ctm_bond_energy(T_(A), T_(B), env, T_(hop), ctm.CTM_BOND_V),
           "eH_ref": O.bond_energy(e, A, B, hop, "H")[0], "eV_ref": O.bond_energy(e, A, B, hop, "V")[0]}
    if e2 is not None:
        out["norm_pert"] = O.norm_2x2(e2, A, B)
        out["eH_pert"] = O.bond_energy(e2, A, B, hop, "H")[0]
    return out


@pytest.mark.parametrize("name,n_iter", [("tiny", 1), ("c2_dl", 20)])
@pytest.mark.parametrize("svd", SVDS)
def test_iterations_gauge_invariant_1e9(name, n_iter, svd):
    """Well-conditioned cases: 2x2 norm and bond energies after n_iter CTM iterations
    (left, right, up, down moves) agree with the oracle within 1e-9 relative."""
    r = _iterate_both(name, n_iter, svd=svd)
    print(name, svd, r)
    assert abs(r["norm_gpu"] - r["norm_ref"]) <= 1e-9 * abs(r["norm_ref"])
    for k in ("eH", "eV"):
        assert abs(r[k + "_gpu"] - r[k + "_ref"]) <= 1e-9 * max(abs(r[k + "_ref"]), 1e-3)


@pytest.mark.parametrize("bond", ["H", "V"])
@pytest.mark.parametrize("name", ["tiny", "c2"])
def test_bond_energy_closure(name, bond):
    """ctm_bond_energy (GPU closure) vs the oracle closure on the same environment."""
    cfg = ci.CONFIGS[name]
    g = ci.generate(cfg)
    h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi)
    env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
    hop = ci.heisenberg_h()
    rho = torch.zeros((cfg.d,) * 4, dtype=torch.float64, device=DEV)
    e = h.ctm_bond_energy(T_(g["A"]), T_(g["B"]), env, T_(hop), ctm.CTM_BOND_H if bond == "H" else ctm.CTM_BOND_V,
                          rho_out=rho)
    e_ref, m_ref = O.bond_energy({"C": g["C"], "T": g["T"]}, g["A"], g["B"], hop, bond)
    assert abs(e - e_ref) <= 1e-10 * max(1.0, abs(e_ref))
    assert np.allclose(rho.cpu().numpy().reshape(4, 4), m_ref, atol=1e-10)


def test_bond_energy_D1_closed_form():
    cfg = ci.custom(2, 1, 3, seed_index=37)
    g = ci.generate(cfg)
    h = ctm.CtmHandle(2, 1, 3)
    env = ctm.Env.from_host(g["C"], g["T"], 1, 3)
    hop = ci.heisenberg_h()
    a, b = g["A"].ravel(), g["B"].ravel()
    ab = np.kron(a, b)
    want = ab @ hop.reshape(4, 4) @ ab / (a @ a) / (b @ b)
    for bond in (ctm.CTM_BOND_H, ctm.CTM_BOND_V):
        e = h.ctm_bond_energy(T_(g["A"]), T_(g["B"]), env, T_(hop), bond)
        assert abs(e - want) <= 1e-12


# ----------------------------------------------------------------------------------------
# REDUCED strategy (Fig 3(a,b)): exact reduced environment and the
# one-shot 4-leg isometry on the GPU
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("d,D,chi", [(2, 2, 8), (2, 4, 32), (2, 3, 20), (2, 6, 64)])
def test_reduced_env_exact(d, D, chi):
    """M_exact (gauge-free: its legs are existing bonds) entrywise against the oracle."""
    cfg = ci.custom(d, D, chi, seed_index=300 + chi, decaying=D >= 6)
    g = ci.generate(cfg)
    C, T, A = g["C"], g["T"], g["A"]
    x = "b"
    M_ref = O.reduced_env_exact(C[(x, 1)], T[(x, 2)], C[(x, 2)], T[(x, 1)], A, A, T[(x, 3)])
    h = ctm.CtmHandle(d, D, chi)
    M = torch.empty((chi, D, D, chi), dtype=torch.float64, device=DEV)
    h.ctm_reduced_env(T_(C[(x, 1)]), T_(T[(x, 2)]), T_(C[(x, 2)]), T_(T[(x, 1)]), T_(A), T_(A), T_(T[(x, 3)]), M,
                      mode=ctm.CTM_RENV_EXACT)
    assert rel_err(M.cpu().numpy(), M_ref) <= 1e-11


STRATS = {"reduced": "CTM_REDUCED_EXACT", "standard": "CTM_STANDARD"}


@pytest.mark.parametrize("strategy", ["reduced", "standard"])
def test_reduced_move_without_truncation_matches_oracle(strategy):
    """No truncation (chi0 = 1 -> 4 -> 16, every isometry square): the REDUCED and STANDARD
    moves are exact."""
    cfg = ci.custom(2, 2, 16, chi0=1, seed_index=22)
    g = ci.generate(cfg)
    h = ctm.CtmHandle(2, 2, 16, flags=ctm.CTM_FLAG_MOVE_ONLY, strategy=getattr(ctm, STRATS[strategy]))
    env = ctm.Env.from_host(g["C"], g["T"], 2, 16)
    h.ctm_left_move(T_(g["A"]), T_(g["B"]), env)
    got = env.to_host()
    ref = O.left_move({"C": g["C"], "T": g["T"]}, g["A"], g["B"], 16, strategy=strategy)
    for x in ("a", "b"):
        y = O.OTHER[x]

        def col(e):
            c = np.einsum("xR,yklx,zmny,Sz->RklmnS", e["C"][(x, 1)], e["T"][(x, 1)], e["T"][(y, 1)], e["C"][(y, 4)])
            return c / np.linalg.norm(c)
        assert np.allclose(col(got), col(ref), atol=1e-12)


@pytest.mark.parametrize("strategy,name", [("reduced", "tiny"), ("reduced", "c2_dl"), ("reduced", "c3_dl"),
                                           ("standard", "tiny"), ("standard", "c2_dl")])
def test_reduced_move_gauge_invariant(strategy, name):
    """One REDUCED / STANDARD left move: the 2x2 norm of the new environment (a
    gauge-invariant closure, evaluated by the oracle on both) agrees with the oracle's move
    of the same strategy."""
    cfg = ci.CONFIGS[name]
    g = ci.generate(cfg, ci.ENV_INIT.get(name))
    A, B = g["A"], g["B"]
    h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, flags=ctm.CTM_FLAG_MOVE_ONLY, strategy=getattr(ctm, STRATS[strategy]))
    env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
    st = h.ctm_left_move(T_(A), T_(B), env)
    assert st["n_svd"] == 4
    ref = O.left_move({"C": g["C"], "T": g["T"]}, A, B, cfg.chi, strategy=strategy)
    n_gpu = O.norm_2x2(env.to_host(), A, B)
    n_ref = O.norm_2x2(ref, A, B)
    assert abs(n_gpu - n_ref) <= 1e-9 * abs(n_ref)


# ----------------------------------------------------------------------------------------
# convergence loop (reading R22): corner spectra on the GPU vs the oracle
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("max_iter,tol,want_iters", [(3, 0.0, 3), (10, 0.06, 2)])
def test_converge_matches_oracle(max_iter, tol, want_iters):
    cfg = ci.CONFIGS["c2_dl"]
    g = ci.generate(cfg)
    A, B = g["A"], g["B"]
    h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi)
    env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
    it, delta, _ = h.ctm_converge(T_(A), T_(B), env, max_iter, tol)
    ref_env, it_ref, delta_ref = O.converge({"C": g["C"], "T": g["T"]}, A, B, cfg.chi, tol, max_iter)
    assert it == it_ref == want_iters
    assert abs(delta - delta_ref) <= 1e-8 * abs(delta_ref)
    n_gpu = O.norm_2x2(env.to_host(), A, B)
    n_ref = O.norm_2x2(ref_env, A, B)
    assert abs(n_gpu - n_ref) <= 1e-9 * abs(n_ref)


@pytest.mark.parametrize("name", ["tiny", "c2"])
def test_site_spins(name):
    """ctm_site_spins (GPU closure) vs the oracle on the same environment."""
    cfg = ci.CONFIGS[name]
    g = ci.generate(cfg)
    h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi)
    env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
    (sa, sb), ms = h.ctm_site_spins(T_(g["A"]), T_(g["B"]), env)
    ref = O.site_spins({"C": g["C"], "T": g["T"]}, g["A"], g["B"])
    assert np.allclose(np.array([sa, sb]), np.array(ref), atol=1e-10, rtol=1e-10)
    assert ms == pytest.approx(O.staggered_magnetization({"C": g["C"], "T": g["T"]}, g["A"], g["B"]), rel=1e-10)


# ----------------------------------------------------------------------------------------
# error conventions on the device path (status codes, no exception across the ABI)
# ----------------------------------------------------------------------------------------
def test_errors_are_status_codes():
    cfg = ci.CONFIGS["tiny"]
    g = ci.generate(cfg)
    h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, flags=ctm.CTM_FLAG_MOVE_ONLY)
    env = ctm.Env.from_host(g["C"], g["T"], cfg.D, cfg.chi)
    L = ctm.lib()
    # null site pointer -> CTM_E_ARG with a message
    assert L.ctm_left_move(h.h, None, None, ctypes_byref(env), None, None, None) == ctm.CTM_E_ARG
    assert b"null" in L.ctm_last_error(h.h)
    # boundary extent above chi -> CTM_E_ARG
    env.c.ext[0][4][0] = cfg.chi + 1
    with pytest.raises(ctm.CtmError) as ei:
        h.ctm_left_move(T_(g["A"]), T_(g["B"]), env)
    assert ei.value.code == ctm.CTM_E_ARG
    env.c.ext[0][4][0] = cfg.chi
    # iso_in / iso_out with the REDUCED strategy -> CTM_E_UNSUPPORTED
    hr = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, flags=ctm.CTM_FLAG_MOVE_ONLY, strategy=ctm.CTM_REDUCED_EXACT)
    iso = torch.zeros(h.iso_numel(), dtype=torch.float64, device=DEV)
    with pytest.raises(ctm.CtmError) as ei:
        hr.ctm_left_move(T_(g["A"]), T_(g["B"]), env, iso_out=iso)
    assert ei.value.code == ctm.CTM_E_UNSUPPORTED
    # the handle is still usable after an error
    h.ctm_left_move(T_(g["A"]), T_(g["B"]), env)


@pytest.mark.parametrize("name,svd", [("tiny", "iso"), ("c2", "iso"), ("c2", "gesvdp")])
def test_non_finite_input_is_reported(name, svd):
    """CHECK_FINITE: a NaN in the environment surfaces as CTM_E_NONFINITE / CTM_E_SOLVER
    (S:L75), never as an illegal access or silently corrupted tensors."""
    cfg = ci.CONFIGS[name]
    g = ci.generate(cfg)
    C = dict(g["C"])
    C[("a", 1)] = C[("a", 1)].copy()
    C[("a", 1)][0, 0] = np.nan
    h = ctm.CtmHandle(cfg.d, cfg.D, cfg.chi, flags=ctm.CTM_FLAG_MOVE_ONLY | ctm.CTM_FLAG_CHECK_FINITE,
                      svd_algo=svd_algo(svd))
    env = ctm.Env.from_host(C, g["T"], cfg.D, cfg.chi)
    with pytest.raises(ctm.CtmError) as ei:
        h.ctm_left_move(T_(g["A"]), T_(g["B"]), env)
    assert ei.value.code in (ctm.CTM_E_NONFINITE, ctm.CTM_E_SOLVER)


def test_chi_p_above_chi_D_is_clamped_with_a_warning():
    """chi' > chi D is clamped to chi D, reported as CTM_W_CLAMPED."""
    h = ctm.CtmHandle(2, 2, 4, chi_p=100, flags=ctm.CTM_FLAG_MOVE_ONLY)
    assert h.clamped


def ctypes_byref(env):
    import ctypes
    return ctypes.byref(env.c)

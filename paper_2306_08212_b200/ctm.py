"""Thin ctypes binding of libctm (include/ctm.h): argument marshalling only.

Every step of the CTMRG move runs in libctm's CUDA kernels / cuSOLVER on the device.
There is no CPU fallback: if libctm.so is missing or no CUDA device is present, the
calls raise.  PyTorch is used only for device memory and streams.

Names follow the C ABI (ctm_init, ctm_reduced_env, ctm_absorb_truncate, ctm_left_move,
ctm_norm_2x2, ctm_bond_energy, ...); `CtmHandle` / `Env` are conveniences around them.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, byref, c_double, c_int, c_int64, c_size_t, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
# CTM_LIB_PATH: A/B experiments against another build of the same ABI (tools only)
LIB_PATH = os.environ.get("CTM_LIB_PATH") or os.path.join(HERE, "libctm.so")

CTM_OK = 0
CTM_W_CLAMPED = 100
CTM_SEQUENTIAL, CTM_REDUCED_EXACT, CTM_STANDARD = 0, 1, 2
CTM_SVD_GESVDP, CTM_SVD_GESVDJ, CTM_SVD_GESVD, CTM_SVD_GRAM, CTM_SVD_ISO = 0, 1, 2, 3, 4
CTM_FLAG_CHECK_FINITE = 1
CTM_FLAG_MOVE_ONLY = 2
CTM_FLAG_PROFILE = 4
CTM_FLAG_WARM_START = 8
CTM_RENV_APPROX, CTM_RENV_EXACT = 0, 1
CTM_BOND_H, CTM_BOND_V = 0, 1
CTM_BOND_H1, CTM_BOND_V1, CTM_BOND_H2, CTM_BOND_V2 = 0, 1, 2, 3
BONDS = {"H1": CTM_BOND_H1, "V1": CTM_BOND_V1, "H2": CTM_BOND_H2, "V2": CTM_BOND_V2}
CTM_TS_SVD, CTM_TS_BASIS = 0, 1
DIRS = {"left": 0, "right": 1, "up": 2, "down": 3}
CTM_E_ARG, CTM_E_CUDA, CTM_E_SOLVER, CTM_E_NONFINITE, CTM_E_NOMEM, CTM_E_UNSUPPORTED = 1, 2, 3, 4, 5, 6
STATUS = {0: "CTM_OK", 1: "CTM_E_ARG", 2: "CTM_E_CUDA", 3: "CTM_E_SOLVER", 4: "CTM_E_NONFINITE",
          5: "CTM_E_NOMEM", 6: "CTM_E_UNSUPPORTED"}


class CtmError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class ctm_params(ctypes.Structure):
    _fields_ = [("d", c_int), ("D", c_int), ("chi", c_int), ("chi_p", c_int), ("chi_pp", c_int),
                ("strategy", c_int), ("svd_algo", c_int), ("svd_tol", c_double), ("flags", c_int)]


class ctm_env(ctypes.Structure):
    _fields_ = [("C", (c_void_p * 4) * 2), ("T", (c_void_p * 4) * 2), ("ext", ((c_int * 2) * 8) * 2)]


class ctm_move_stats(ctypes.Structure):
    _fields_ = [("ms_total", c_double), ("ms_svd", c_double), ("ms_contract", c_double), ("flops", c_double),
                ("min_gap", c_double), ("n_svd", c_int), ("n_kernels", c_int), ("ms_gemm", c_double),
                ("gemm_flops", c_double), ("gemm_launches", c_int), ("ms_isometry", c_double),
                ("n_svd_fallback", c_int), ("ms_jacobi", c_double), ("jacobi_flops", c_double),
                ("n_jacobi", c_int), ("jacobi_cta_ms", c_double),
                ("cut_gap", (c_double * 2) * 2), ("side_gap", (c_double * 4) * 2),
                ("ms_commit", c_double), ("commit_bytes", c_double), ("n_commit", c_int),
                ("n_warm", c_int), ("n_warm_hit", c_int), ("n_warm_retry", c_int)]

    def as_dict(self):
        out = {}
        for k, _ in self._fields_:
            v = getattr(self, k)
            out[k] = [list(r) for r in v] if k in ("cut_gap", "side_gap") else v
        return out


_lib = None


def lib():
    """Load libctm.so (fails loudly: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libctm.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        P = c_void_p
        sig = {
            "ctm_abi_version": (c_int, []),
            "ctm_init": (c_int, [POINTER(c_void_p), POINTER(ctm_params), c_uint64, POINTER(c_size_t)]),
            "ctm_set_workspace": (c_int, [P, P, c_size_t]),
            "ctm_set_stream": (c_int, [P, c_uint64]),
            "ctm_destroy": (c_int, [P]),
            "ctm_last_error": (ctypes.c_char_p, [P]),
            "ctm_reduced_env": (c_int, [P, P, P, P, P, P, P, P, c_int, P, P, P]),
            "ctm_absorb_truncate": (c_int, [P, P, P, P, P, P, P, P, P]),
            "ctm_left_move": (c_int, [P, P, P, POINTER(ctm_env), P, P, POINTER(ctm_move_stats)]),
            "ctm_move": (c_int, [P, c_int, P, P, POINTER(ctm_env), P, POINTER(ctm_move_stats)]),
            "ctm_ts_isometry": (c_int, [P, P, c_int, c_int, c_int, c_int, c_int, c_int, c_int, P, P,
                                        POINTER(c_double)]),
            "ctm_iterate": (c_int, [P, P, P, POINTER(ctm_env), c_int, POINTER(ctm_move_stats)]),
            "ctm_converge": (c_int, [P, P, P, POINTER(ctm_env), c_int, c_double, POINTER(c_int), POINTER(c_double),
                                     POINTER(ctm_move_stats)]),
            "ctm_norm_2x2": (c_int, [P, P, P, POINTER(ctm_env), POINTER(c_double), POINTER(c_double)]),
            "ctm_site_spins": (c_int, [P, P, P, POINTER(ctm_env), POINTER(c_double)]),
            "ctm_bond_energy": (c_int, [P, P, P, POINTER(ctm_env), P, c_int, P, POINTER(c_double)]),
            "ctm_move_flops": (c_double, [c_int, c_int, c_int, c_int, c_int]),
            "ctm_trotter_gate": (c_int, [P, P, c_double, P]),
            "ctm_bond_update": (c_int, [P, P, P, POINTER(ctm_env), P, c_int, c_int, P, P, POINTER(c_double)]),
            "ctm_trotter_step": (c_int, [P, P, P, POINTER(ctm_env), P, c_double, c_int, c_int, POINTER(c_double)]),
            "ctm_kernel_count": (c_int64, [P]),
            "ctm_warm_reset": (c_int, [P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return ["ctm_abi_version", "ctm_init", "ctm_set_workspace", "ctm_set_stream", "ctm_destroy",
            "ctm_last_error", "ctm_reduced_env", "ctm_ts_isometry", "ctm_absorb_truncate", "ctm_left_move", "ctm_move",
            "ctm_iterate", "ctm_converge", "ctm_site_spins", "ctm_norm_2x2", "ctm_bond_energy", "ctm_move_flops", "ctm_kernel_count",
            "ctm_trotter_gate", "ctm_bond_update", "ctm_trotter_step", "ctm_warm_reset"]


def ctm_move_flops(d, D, chi, chi_p=None, chi_pp=None):
    return lib().ctm_move_flops(d, D, chi, chi if chi_p is None else chi_p, chi if chi_pp is None else chi_pp)


def _ptr(t):
    if t is None:
        return None
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise TypeError("expected a contiguous float64 CUDA tensor")
    return c_void_p(t.data_ptr())


class CtmHandle:
    """Owns a ctm_handle and its torch-allocated workspace."""

    def __init__(self, d, D, chi, chi_p=None, chi_pp=None, svd_algo=CTM_SVD_ISO, flags=0,
                 svd_tol=0.0, stream=None, device="cuda", strategy=None):
        import torch
        self.torch = torch
        if not torch.cuda.is_available():
            raise RuntimeError("libctm needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.params = ctm_params(d, D, chi, chi if chi_p is None else chi_p, chi if chi_pp is None else chi_pp,
                                 CTM_SEQUENTIAL if strategy is None else strategy, svd_algo, svd_tol, flags)
        h = c_void_p()
        ws = c_size_t()
        with torch.cuda.device(self.device):   # the handle lives on (and records) this device
            rc = lib().ctm_init(byref(h), byref(self.params), self.stream.cuda_stream, byref(ws))
        if rc not in (CTM_OK, CTM_W_CLAMPED):
            raise CtmError(rc, "ctm_init failed")
        self.clamped = rc == CTM_W_CLAMPED
        self.h = h
        self.ws_bytes = ws.value
        self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self._check(lib().ctm_set_workspace(self.h, c_void_p(self.workspace.data_ptr()), self.ws_bytes))

    def _check(self, rc):
        if rc != CTM_OK:
            raise CtmError(rc, lib().ctm_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            lib().ctm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def kernel_count(self):
        return lib().ctm_kernel_count(self.h)

    def ctm_warm_reset(self):
        self._check(lib().ctm_warm_reset(self.h))

    # --- ABI calls --------------------------------------------------------------------
    def ctm_absorb_truncate(self, T, X, Xbra, v1_in, v2_in, v1_out, v2_out, T_out):
        self._check(lib().ctm_absorb_truncate(self.h, _ptr(T), _ptr(X), _ptr(Xbra), _ptr(v1_in), _ptr(v2_in),
                                              _ptr(v1_out), _ptr(v2_out), _ptr(T_out)))
        return T_out

    def ctm_reduced_env(self, C1, T2, C2, T1, X, Xbra, T3, M_out, iso_out=None, mode=CTM_RENV_APPROX, iso_in=None):
        self._check(lib().ctm_reduced_env(self.h, _ptr(C1), _ptr(T2), _ptr(C2), _ptr(T1), _ptr(X), _ptr(Xbra),
                                          _ptr(T3), mode, _ptr(M_out), _ptr(iso_in), _ptr(iso_out)))
        return M_out

    def ctm_left_move(self, A, B, env, iso_in=None, iso_out=None, stats=True):
        """stats=False passes no stats struct: the call then never synchronises the stream
        (with iso_in and without CTM_FLAG_CHECK_FINITE it is capturable in a CUDA graph)."""
        st = ctm_move_stats()
        self._check(lib().ctm_left_move(self.h, _ptr(A), _ptr(B), byref(env.c), _ptr(iso_in), _ptr(iso_out),
                                        byref(st) if stats else None))
        return st.as_dict() if stats else None

    def ctm_move(self, direction, A, B, env, iso_out=None):
        st = ctm_move_stats()
        self._check(lib().ctm_move(self.h, DIRS[direction], _ptr(A), _ptr(B), byref(env.c), _ptr(iso_out),
                                   byref(st)))
        return st.as_dict()

    def ctm_ts_isometry(self, Q, c1, c2, mode=CTM_TS_BASIS):
        """TS(Q; c1, c2) on a (P, K, B, F) device tensor -> (v1, v2, (gap1, gap2))."""
        P_, K, B, F = Q.shape
        n1 = min(c1, P_ * K)
        n2 = min(c2, n1 * B)
        torch = self.torch
        v1 = torch.empty((P_, K, n1), dtype=torch.float64, device=Q.device)
        v2 = torch.empty((n1, B, n2), dtype=torch.float64, device=Q.device)
        gaps = (c_double * 2)()
        self._check(lib().ctm_ts_isometry(self.h, _ptr(Q), P_, K, B, F, c1, c2, mode, _ptr(v1), _ptr(v2), gaps))
        return v1, v2, (gaps[0], gaps[1])

    def ctm_converge(self, A, B, env, max_iter, tol):
        """Returns (iterations, last corner-spectrum distance, stats dict)."""
        st = ctm_move_stats()
        it = c_int()
        delta = c_double()
        self._check(lib().ctm_converge(self.h, _ptr(A), _ptr(B), byref(env.c), max_iter, tol, byref(it), byref(delta),
                                       byref(st)))
        return it.value, delta.value, st.as_dict()

    def ctm_site_spins(self, A, B, env):
        """((Sx_A, Sz_A), (Sx_B, Sz_B)) and m_s = (|<S>_A| + |<S>_B|) / 2."""
        o = (c_double * 5)()
        self._check(lib().ctm_site_spins(self.h, _ptr(A), _ptr(B), byref(env.c), o))
        return ((o[0], o[1]), (o[2], o[3])), o[4]   # m_s computed on the device (out[4])

    def ctm_iterate(self, A, B, env, n_iter):
        st = ctm_move_stats()
        self._check(lib().ctm_iterate(self.h, _ptr(A), _ptr(B), byref(env.c), n_iter, byref(st)))
        return st.as_dict()

    def ctm_norm_2x2(self, A, B, env):
        v, r = c_double(), c_double()
        self._check(lib().ctm_norm_2x2(self.h, _ptr(A), _ptr(B), byref(env.c), byref(v), byref(r)))
        return v.value, r.value

    def ctm_bond_energy(self, A, B, env, h, bond=CTM_BOND_H, rho_out=None):
        e = c_double()
        self._check(lib().ctm_bond_energy(self.h, _ptr(A), _ptr(B), byref(env.c), _ptr(h), bond, _ptr(rho_out),
                                          byref(e)))
        return e.value

    # --- imaginary-time evolution -----------------------------------
    def ctm_trotter_gate(self, hop, delta):
        """exp(-delta h) on the device (d,d,d,d)."""
        g = self.torch.empty_like(hop)
        self._check(lib().ctm_trotter_gate(self.h, _ptr(hop), delta, _ptr(g)))
        return g

    def ctm_bond_update(self, A, B, env, gate, bond, sweeps, A_out=None, B_out=None):
        """One FFU bond update (bond in 'H1','H2','V1','V2'); returns (A', B', (cost, tNt))."""
        A_out = self.torch.empty_like(A) if A_out is None else A_out
        B_out = self.torch.empty_like(B) if B_out is None else B_out
        c = (c_double * 2)()
        self._check(lib().ctm_bond_update(self.h, _ptr(A), _ptr(B), byref(env.c), _ptr(gate), BONDS[bond], sweeps,
                                          _ptr(A_out), _ptr(B_out), c))
        return A_out, B_out, (c[0], c[1])

    def ctm_trotter_step(self, A, B, env, hop, delta, sweeps, refresh=True):
        """One second-order Trotter step, A and B updated in place; returns 7 (cost, tNt)."""
        c = (c_double * 14)()
        self._check(lib().ctm_trotter_step(self.h, _ptr(A), _ptr(B), byref(env.c), _ptr(hop), delta, sweeps,
                                           1 if refresh else 0, c))
        return [(c[2 * i], c[2 * i + 1]) for i in range(7)]

    def iso_numel(self):
        p = self.params
        return 2 * 2 * (p.chi * p.D * p.chi_p + p.chi_p * p.D * p.chi)


class Env:
    """The 16 environment tensors in device buffers of capacity chi (ctm_env)."""

    SUBS = ("a", "b")

    def __init__(self, D, chi, device="cuda"):
        import torch
        self.D, self.chi = D, chi
        self.C = {(x, k): torch.zeros(chi * chi, dtype=torch.float64, device=device)
                  for x in self.SUBS for k in (1, 2, 3, 4)}
        self.T = {(x, k): torch.zeros(chi * D * D * chi, dtype=torch.float64, device=device)
                  for x in self.SUBS for k in (1, 2, 3, 4)}
        self.c = ctm_env()
        for xi, x in enumerate(self.SUBS):
            for k in (1, 2, 3, 4):
                self.c.C[xi][k - 1] = self.C[(x, k)].data_ptr()
                self.c.T[xi][k - 1] = self.T[(x, k)].data_ptr()
                self.c.ext[xi][k - 1][0] = self.c.ext[xi][k - 1][1] = chi
                self.c.ext[xi][4 + k - 1][0] = self.c.ext[xi][4 + k - 1][1] = chi

    def ext(self, kind, x, k):
        xi = self.SUBS.index(x)
        j = (k - 1) + (4 if kind == "T" else 0)
        return self.c.ext[xi][j][0], self.c.ext[xi][j][1]

    @classmethod
    def from_host(cls, C, T, D, chi, device="cuda", non_blocking=False):
        """C, T: dicts {(x,k): numpy array} in clockwise storage order."""
        import torch
        env = cls(D, chi, device)
        for xi, x in enumerate(cls.SUBS):
            for k in (1, 2, 3, 4):
                c, t = C[(x, k)], T[(x, k)]
                env.C[(x, k)][: c.size].copy_(torch.from_numpy(c.reshape(-1)), non_blocking=non_blocking)
                env.T[(x, k)][: t.size].copy_(torch.from_numpy(t.reshape(-1)), non_blocking=non_blocking)
                env.c.ext[xi][k - 1][0], env.c.ext[xi][k - 1][1] = c.shape
                env.c.ext[xi][4 + k - 1][0], env.c.ext[xi][4 + k - 1][1] = t.shape[0], t.shape[3]
        return env

    def to_host(self):
        C, T = {}, {}
        for x in self.SUBS:
            for k in (1, 2, 3, 4):
                e0, e1 = self.ext("C", x, k)
                C[(x, k)] = self.C[(x, k)][: e0 * e1].cpu().numpy().reshape(e0, e1)
                e0, e1 = self.ext("T", x, k)
                T[(x, k)] = self.T[(x, k)][: e0 * self.D * self.D * e1].cpu().numpy().reshape(e0, self.D, self.D, e1)
        return {"C": C, "T": T}

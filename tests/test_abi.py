"""CPU-side checks of the C-ABI library: it loads and exports every symbol include/ctm.h
declares (no compute calls without a GPU), and host-only entry points behave."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ctm.h")
LIB = os.path.join(ROOT, "paper_2306_08212_b200", "libctm.so")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ctm_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2306_08212_b200 import build
        build.build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_six_north_star_calls():
    names = _declared()
    for n in ("ctm_init", "ctm_reduced_env", "ctm_absorb_truncate", "ctm_left_move", "ctm_norm_2x2",
              "ctm_bond_energy"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for n in _declared():
        assert hasattr(lib, n), n


def test_binding_covers_header():
    from paper_2306_08212_b200 import ctm
    assert set(_declared()) <= set(ctm.exported_symbols())


def test_abi_version_and_flops(lib):
    from paper_2306_08212_b200 import ctm
    assert ctm.lib().ctm_abi_version() == 3
    # F_move = 147.9 GF at d=2, D=8, chi=128
    f = ctm.ctm_move_flops(2, 8, 128)
    assert abs(f / 1e9 - 147.9) < 0.1
    # closed form of SURVEY 8(a)
    d, D, c = 2, 8, 128
    chain = 4 * c**3 * D**3 + 4 * d * c**3 * D**3 + 4 * d * c**2 * D**5
    corner = 2 * c**3 * D**2 + 4 * c**3 * D
    renv = chain + 14 * c**3 * D**2 + 4 * c**3 * D
    assert abs(f - 2 * (2 * renv + 2 * chain + 4 * corner)) < 1e-6 * f


def test_null_handle_is_an_argument_error(lib):
    from paper_2306_08212_b200 import ctm
    L = ctm.lib()
    assert L.ctm_destroy(None) == 1
    assert L.ctm_left_move(None, None, None, None, None, None, None) == 1
    assert L.ctm_last_error(None) == b"null handle"


def test_init_rejects_bad_sizes(lib):
    from paper_2306_08212_b200 import ctm
    h = ctypes.c_void_p()
    ws = ctypes.c_size_t()
    p = ctm.ctm_params(2, 0, 8, 8, 8, 0, 0, 0.0, 0)
    assert ctm.lib().ctm_init(ctypes.byref(h), ctypes.byref(p), 0, ctypes.byref(ws)) == 1
    p = ctm.ctm_params(2, 2, 8, 8, 8, 7, 0, 0.0, 0)   # unknown strategy
    assert ctm.lib().ctm_init(ctypes.byref(h), ctypes.byref(p), 0, ctypes.byref(ws)) == 6

"""B200-native CTMRG move of arXiv 2306.08212 (reduced environment + sequential order).

The product is libctm.so (include/ctm.h); `paper_2306_08212_b200.ctm` is its thin
ctypes binding.  Build with `python -m paper_2306_08212_b200.build` or
`__graft_entry__.build()`."""
from . import ctm  # noqa: F401
from .ctm import CtmHandle, Env, CtmError  # noqa: F401

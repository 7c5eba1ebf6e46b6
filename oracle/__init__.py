"""CPU float64 oracle (TEST INFRASTRUCTURE ONLY; see oracle/ctm_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs.  The product package never imports it."""
from . import ctm_oracle  # noqa: F401

"""ORACLE -- test infrastructure, NOT part of the product path.

A plain, slow, fp64 CPU implementation of DiffXPBD's forward XPBD substep and
analytic adjoint backward pass, written from PAPER.md (arxiv 2301.01396), each
function citing the passage it follows.  It shares no code with the CUDA path
(`paper_2301_01396_b200/`) and neither imports the other.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` leg may import, call, link or execute anything under
`oracle/`.  The product (C-ABI library + binding) fails loudly when its CUDA
extension is missing; it never falls back to this code.

Pins: see tests/test_oracle_*.py and DESIGN.md section "Oracle pins".  Every
function here is pinned (no "parity unpinned" entries at present).
"""
from .coloring import greedy_color, greedy_color_py  # noqa: F401
from . import constraints  # noqa: F401
from .xpbd import OracleModel  # noqa: F401

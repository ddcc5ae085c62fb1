"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct fp64 CPU implementation (numpy) of what the
MGRIT/Parareal hot path computes, written from PAPER.md (arXiv:1910.03726).
Every function cites the passage it follows ("P:n" = PAPER.md line n).

Rules (DESIGN.md §"Oracle"):
* Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
  `--impl reference` legs may import anything under `oracle/`.
* It shares no code with the CUDA path (`paper_1910_03726_b200/`): neither
  imports the other.  The only common module is `workloads/` (seeded input
  generators, none of the method's arithmetic).
* It follows the paper's definitions step by step over the FULL space-time
  state; library primitives (np.roll, np.fft, np.linalg) serve as steps only.

Parity pins live in tests/test_oracle_*.py (run with `-m "not gpu"`).
Parity unpinned: the paper's own Psi coefficients and per-level sparsity
patterns (shown only in figures), its RNG stream, and XBraid cycle details
(DESIGN.md §"Readings").
"""
from . import discretization, mgrit, psi, theory  # noqa: F401

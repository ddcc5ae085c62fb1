"""Oracle: MGRIT / Parareal on the FULL space-time state.

ORACLE — test infrastructure only (see oracle/__init__.py).

Follows PAPER.md §2.2 step by step:
* space-time system U[n+1] = Phi U[n], U[0] = u0, block lower bidiagonal;
* C-points n = j m, F-points otherwise;
* F-relaxation: step from each C-point across its F-interval;
* C-relaxation: step from the last F-point to the next C-point;
* FCF = F, C, F (used "exclusively");
* coarse error equation e^{n+1} = Psi e^n + r^{n+1}, e^0 = 0, with r the fine
  residual injected at the C-points;
* correction at C-points + "ideal interpolation" = injection + F-relaxation;
* recursion on the coarse problem = multilevel V-cycle,
  sequential solve on the coarsest level;
* stopping: space-time residual < 1e-10 in the discrete L2 norm,
  norm = sqrt(dx*dt*sum r^2) (R1-Q1), counted after each iteration (R2).

Level-l equations are written in right-hand-side form (R12):
    U[0] = g[0],   U[n+1] = Phi_l U[n] + g[n+1]
with g_1 = (u0, 0, ..., 0) on the fine level and U_l = 0 as the initial guess
of every coarser level (error-correction form).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np


# --------------------------------------------------------------------------
# Relaxation sweeps on one level, with RHS g (g = None means g = 0
# except row 0).  All intervals are independent; numpy steps them together
# (the same arithmetic per point as one interval at a time).
# --------------------------------------------------------------------------
def f_relax(U: np.ndarray, phi: Callable, m: int, g: Optional[np.ndarray] = None) -> None:
    """U[jm+i] = Phi U[jm+i-1] (+ g[jm+i]),  i = 1..m-1, every interval j."""
    nt = U.shape[0] - 1
    for i in range(1, m):
        rows = np.arange(i, nt, m)              # F-points jm+i
        U[rows] = phi(U[rows - 1])
        if g is not None:
            U[rows] = U[rows] + g[rows]


def c_relax(U: np.ndarray, phi: Callable, m: int, g: Optional[np.ndarray] = None) -> None:
    """U[(j+1)m] = Phi U[(j+1)m-1] (+ g[(j+1)m]), every C-point except t = 0."""
    nt = U.shape[0] - 1
    rows = np.arange(m, nt + 1, m)
    U[rows] = phi(U[rows - 1])
    if g is not None:
        U[rows] = U[rows] + g[rows]


def residual_rows(U: np.ndarray, phi: Callable, rows: np.ndarray,
                  g: Optional[np.ndarray] = None) -> np.ndarray:
    """r[n] = g[n] + Phi U[n-1] - U[n] at the given rows n >= 1."""
    r = phi(U[rows - 1]) - U[rows]
    if g is not None:
        r = g[rows] + r
    return r


def residual_norm(U: np.ndarray, phi: Callable, dx: float, dt: float,
                  g: Optional[np.ndarray] = None) -> float:
    """Discrete L2 space-time residual over ALL rows n = 1..nt (R1-Q1)."""
    nt = U.shape[0] - 1
    r = residual_rows(U, phi, np.arange(1, nt + 1), g)
    return float(np.sqrt(dx * dt * np.sum(r * r)))


def sequential_rhs(phi: Callable, g: np.ndarray) -> np.ndarray:
    """Coarsest-level solve U[0] = g[0], U[n+1] = Phi U[n] + g[n+1]."""
    U = np.empty_like(g)
    U[0] = g[0]
    for n in range(g.shape[0] - 1):
        U[n + 1] = phi(U[n]) + g[n + 1]
    return U


# --------------------------------------------------------------------------
# One MGRIT cycle (V-cycle; two-level when len(phis) == 2)
# --------------------------------------------------------------------------
def vcycle(level: int, U: np.ndarray, g: Optional[np.ndarray], phis: Sequence[Callable],
           m: int, relax: str) -> None:
    """V(level, U, g): FCF (or F) relaxation, residual injection, coarse solve
    (recursive, sequential on the coarsest level), correction + F-relaxation
    (P:206-212).  U is modified in place."""
    phi = phis[level]
    nt = U.shape[0] - 1
    if level == len(phis) - 1:                       # coarsest: sequential
        U[:] = sequential_rhs(phi, g if g is not None else _fine_rhs(U))
        return
    # pre-relaxation
    f_relax(U, phi, m, g)
    if relax == "FCF":
        c_relax(U, phi, m, g)
        f_relax(U, phi, m, g)
    # residual at C-points, injected as the coarse right-hand side
    cpts = np.arange(m, nt + 1, m)
    gc = np.zeros((nt // m + 1, U.shape[1]))
    gc[1:] = residual_rows(U, phi, cpts, g)
    # coarse error equation e^{j+1} = Psi e^j + r^{j+1}, e^0 = 0
    E = np.zeros_like(gc)
    vcycle(level + 1, E, gc, phis, m, relax)
    # correction at C-points + ideal interpolation
    U[cpts] = U[cpts] + E[1:]
    f_relax(U, phi, m, g)


def fcycle(level: int, U: np.ndarray, g: Optional[np.ndarray], phis: Sequence[Callable],
           m: int, relax: str) -> None:
    """F(level, U, g): the multigrid F-cycle (P:622, P:843 name it without defining it;
    DESIGN.md R19 reading): relaxation and residual injection as in V, but the coarse
    error equation is solved approximately by one F-cycle followed by one V-cycle on the
    coarse level, both from e = 0 / the F-cycle's result; then correction + F-relaxation.
    On the coarsest level it is the sequential solve.  U is modified in place."""
    phi = phis[level]
    nt = U.shape[0] - 1
    if level == len(phis) - 1:
        U[:] = sequential_rhs(phi, g if g is not None else _fine_rhs(U))
        return
    f_relax(U, phi, m, g)
    if relax == "FCF":
        c_relax(U, phi, m, g)
        f_relax(U, phi, m, g)
    cpts = np.arange(m, nt + 1, m)
    gc = np.zeros((nt // m + 1, U.shape[1]))
    gc[1:] = residual_rows(U, phi, cpts, g)
    E = np.zeros_like(gc)
    fcycle(level + 1, E, gc, phis, m, relax)
    vcycle(level + 1, E, gc, phis, m, relax)
    U[cpts] = U[cpts] + E[1:]
    f_relax(U, phi, m, g)


def _fine_rhs(U):
    g = np.zeros_like(U)
    g[0] = U[0]
    return g


@dataclass
class SolveReport:
    """Iterations K, residual history (K+1 entries), converged flag."""
    iterations: int
    history: List[float]
    converged: bool
    states: List[np.ndarray] = field(default_factory=list)   # C-rows after each iteration
    nonfinite: bool = False


def solve(U: np.ndarray, phis: Sequence[Callable], m: int, dx: float, dt: float,
          relax: str = "FCF", tol: float = 1e-10, max_iter: int = 64,
          keep_states: bool = False, cycle: str = "V",
          on_iter: Optional[Callable[[int, np.ndarray], None]] = None,
          g0: Optional[np.ndarray] = None) -> SolveReport:
    """MGRIT / Parareal iteration on the fine space-time iterate U (in place).

    U[0] holds u0 and is never modified.  The residual is
    measured on the iterate after k complete iterations; K = first k with
    ||r^(k)|| < tol (R2).  No early stop on growth (R15), except
    for non-finite values.  cycle: "V" or "F" (R19).  on_iter(k, U), if
    given, is called after iteration k with the iterate (read-only observation, e.g. to
    sample rows for a golden file; it does not take part in the arithmetic).  g0: the fine
    level's right-hand side (rows 1..nt; row 0 unused) for an affine fine propagator
    U[n+1] = Phi U[n] + g0[n+1], e.g. the inflow forcing of oracle.inflow (R12, R20);
    None = 0."""
    phi = phis[0]
    hist = [residual_norm(U, phi, dx, dt, g0)]
    states = []
    k = 0
    converged = hist[0] < tol
    nonfinite = False
    while not converged and k < max_iter:
        (fcycle if cycle == "F" else vcycle)(0, U, g0, phis, m, relax)
        k += 1
        r = residual_norm(U, phi, dx, dt, g0)
        hist.append(r)
        if keep_states:
            states.append(U[::m].copy())
        if on_iter is not None:
            on_iter(k, U)
        if not np.isfinite(r):
            nonfinite = True
            break
        converged = r < tol
    return SolveReport(k, hist, converged, states, nonfinite)


# --------------------------------------------------------------------------
# Operator complexity, eq. (OC)
# --------------------------------------------------------------------------
def operator_complexity(nnz: Sequence[int], m: int) -> float:
    return sum(m ** (-l) * nnz[l] for l in range(len(nnz))) / nnz[0]

"""Oracle: spatial stencils, Butcher tableaux, the one-step operator Phi.

ORACLE — test infrastructure only (see oracle/__init__.py).

Follows PAPER.md §2.1:
* U1-U5 upwind stencils.
* L = discretisation of -alpha d/dx, periodic => circulant.
* ERK / SDIRK Runge-Kutta schemes, P:135 and Appendix A tableaux P:875-1025.
* One-step form u^{n+1} = Phi u^n.
* CFL number c = alpha dt/dx.

Index convention (R1): a circulant operator A is stored as a stencil
{d: a_d} with (A u)_i = sum_d a_d u_{(i+d) mod nx}.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Dict, List, Sequence

import numpy as np

# ---------------------------------------------------------------------------
# Upwind stencils U1..U5:  u'(x_i) ~ (1/(den dx)) sum_d w_d u_{i+d}
# ---------------------------------------------------------------------------
UPWIND: Dict[int, tuple] = {
    1: ({0: 1, -1: -1}, 1),
    2: ({0: 3, -1: -4, -2: 1}, 2),
    3: ({1: 2, 0: 3, -1: -6, -2: 1}, 6),
    4: ({1: 3, 0: 10, -1: -18, -2: 6, -3: -1}, 12),
    5: ({2: -3, 1: 30, 0: 20, -1: -60, -2: 15, -3: -2}, 60),
}


def z_coefficients(order: int, cfl: float) -> Dict[int, float]:
    """Stencil of Z = dt*L for U_p at CFL number c.

    (dt L u)_i = -(alpha dt/dx)(1/den) sum_d w_d u_{i+d}, so z_d = (-c*w_d)/den.
    The expression order (-c*w)/den is the canonical rounding (R3)."""
    w, den = UPWIND[order]
    return {d: (-cfl * float(wd)) / float(den) for d, wd in sorted(w.items())}


# ---------------------------------------------------------------------------
# Butcher tableaux (Appendix A)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Tableau:
    name: str
    A: tuple            # s x s, row-major tuples
    b: tuple
    c: tuple
    implicit: bool

    @property
    def s(self) -> int:
        return len(self.b)


def _tab(name, A, b, c, implicit=False) -> Tableau:
    A = tuple(tuple(float(x) for x in row) for row in A)
    return Tableau(name, A, tuple(float(x) for x in b), tuple(float(x) for x in c), implicit)


def sdirk3_constants():
    """SDIRK3 constants, P:960-965 (zeta from its printed digits)."""
    zeta = 0.43586652150845899942
    alpha = (1.0 + zeta) / 2.0
    beta = (1.0 - zeta) / 2.0
    gamma = -1.5 * zeta * zeta + 4.0 * zeta - 0.25
    eps = 1.5 * zeta * zeta - 5.0 * zeta + 1.25
    return zeta, alpha, beta, gamma, eps


def tableau(name: str) -> Tableau:
    if name == "erk1":      # Euler
        return _tab(name, [[0.0]], [1.0], [0.0])
    if name == "erk2":      # SSP RK2
        return _tab(name, [[0, 0], [1.0, 0]], [1 / 2, 1 / 2], [0, 1])
    if name == "erk3_ssp":  # SSP RK3
        return _tab(name, [[0, 0, 0], [1.0, 0, 0], [1 / 4, 1 / 4, 0]],
                    [1 / 6, 1 / 6, 2 / 3], [0, 1, 1 / 2])
    if name == "erk3_kutta":  # Kutta's third-order method (BJ cfg2; R6)
        return _tab(name, [[0, 0, 0], [1 / 2, 0, 0], [-1.0, 2.0, 0]],
                    [1 / 6, 2 / 3, 1 / 6], [0, 1 / 2, 1])
    if name == "erk4":      # classical RK4
        return _tab(name, [[0, 0, 0, 0], [1 / 2, 0, 0, 0], [0, 1 / 2, 0, 0], [0, 0, 1.0, 0]],
                    [1 / 6, 1 / 3, 1 / 3, 1 / 6], [0, 1 / 2, 1 / 2, 1])
    if name == "erk5":      # Butcher (236a)
        return _tab(name,
                    [[0, 0, 0, 0, 0, 0],
                     [1 / 4, 0, 0, 0, 0, 0],
                     [1 / 8, 1 / 8, 0, 0, 0, 0],
                     [0, 0, 1 / 2, 0, 0, 0],
                     [3 / 16, -3 / 8, 3 / 8, 9 / 16, 0, 0],
                     [-3 / 7, 8 / 7, 6 / 7, -12 / 7, 8 / 7, 0]],
                    [7 / 90, 0, 32 / 90, 12 / 90, 32 / 90, 7 / 90],
                    [0, 1 / 4, 1 / 4, 1 / 2, 3 / 4, 1])
    if name == "sdirk1":    # backward Euler
        return _tab(name, [[1.0]], [1.0], [1.0], True)
    if name == "sdirk2":
        g = 1.0 - np.sqrt(2.0) / 2.0
        h = np.sqrt(2.0) / 2.0
        return _tab(name, [[g, 0], [h, g]], [h, g], [g, 1.0], True)
    if name == "sdirk3":
        zeta, al, be, ga, ep = sdirk3_constants()
        return _tab(name, [[zeta, 0, 0], [be, zeta, 0], [ga, ep, zeta]], [ga, ep, zeta],
                    [zeta, al, 1.0], True)
    if name == "sdirk4":    # Hairer-Wanner (6.16)
        A = [[1 / 4, 0, 0, 0, 0],
             [1 / 2, 1 / 4, 0, 0, 0],
             [17 / 50, -1 / 25, 1 / 4, 0, 0],
             [371 / 1360, -137 / 2720, 15 / 544, 1 / 4, 0],
             [25 / 24, -49 / 48, 125 / 16, -85 / 12, 1 / 4]]
        return _tab(name, A, A[4], [1 / 4, 3 / 4, 11 / 20, 1 / 2, 1.0], True)
    raise KeyError(name)


# ---------------------------------------------------------------------------
# Circulant stencil application and solve
# ---------------------------------------------------------------------------
def apply_stencil(u: np.ndarray, stencil: Dict[int, float]) -> np.ndarray:
    """(A u)_i = sum_d a_d u_{(i+d) mod nx}, along the last axis, d ascending."""
    out = None
    for d in sorted(stencil):
        term = stencil[d] * np.roll(u, -d, axis=-1)     # roll(u,-d)[i] = u[i+d]
        out = term if out is None else out + term
    return out


def first_column(stencil: Dict[int, float], nx: int) -> np.ndarray:
    """Column 0 of the circulant: entry (j, 0) = a_{-j} (R1)."""
    col = np.zeros(nx)
    for d, a in stencil.items():
        col[(-d) % nx] += a
    return col


def solve_circulant(rhs: np.ndarray, col: np.ndarray) -> np.ndarray:
    """x with C x = rhs for the circulant with first column `col`.

    Circulants are diagonalised by the DFT (Corollary 1 P:154-159)."""
    return np.real(np.fft.ifft(np.fft.fft(rhs, axis=-1) / np.fft.fft(col), axis=-1))


# ---------------------------------------------------------------------------
# The fine propagator Phi (Lemma 1) in Runge-Kutta
# stage form.  DESIGN.md R5: the stage form is the contract (no collapsing).
# ---------------------------------------------------------------------------
class RKPhi:
    """u -> Phi u for a Runge-Kutta scheme applied to du/dt = L u.

    ERK:   k_i = Z (u + sum_{l<i} a_il k_l)
    SDIRK: (I - a_ii Z) y_i = u + sum_{l<i} a_il k_l,  k_i = Z y_i
    Phi u = u + sum_i b_i k_i      (R14: b-form also for SDIRK)
    """

    def __init__(self, order: int, tab: Tableau, cfl: float, nx: int):
        self.order, self.tab, self.cfl, self.nx = order, tab, cfl, nx
        self.z = z_coefficients(order, cfl)
        self.nnz = len(self.z)
        if tab.implicit:
            self._mcols = []
            for i in range(tab.s):
                aii = tab.A[i][i]
                mst = {d: -aii * zd for d, zd in self.z.items()}
                mst[0] = mst.get(0, 0.0) + 1.0
                self._mcols.append(first_column(mst, nx))

    def __call__(self, u: np.ndarray) -> np.ndarray:
        A, b = self.tab.A, self.tab.b
        ks: List[np.ndarray] = []
        for i in range(self.tab.s):
            y = u
            for l in range(i):
                if A[i][l] != 0.0:
                    y = y + A[i][l] * ks[l]
            if self.tab.implicit:
                y = solve_circulant(y, self._mcols[i])
            ks.append(apply_stencil(y, self.z))
        out = u
        for i in range(self.tab.s):
            if b[i] != 0.0:
                out = out + b[i] * ks[i]
        return out


class StencilPhi:
    """u -> Psi u for an explicit circulant stencil Psi."""

    def __init__(self, stencil: Dict[int, float], nx: int):
        self.stencil = dict(sorted(stencil.items()))
        self.nx = nx
        self.nnz = len(stencil)

    def __call__(self, u):
        return apply_stencil(u, self.stencil)


class PowerPhi:
    """u -> Phi^q u (the ideal coarse operator Psi_ideal = Phi^m)."""

    def __init__(self, phi, q: int):
        self.phi, self.q, self.nx = phi, q, phi.nx
        self.nnz = None

    def __call__(self, u):
        for _ in range(self.q):
            u = self.phi(u)
        return u


def make_phi(order: int, tableau_name: str, cfl: float, nx: int) -> RKPhi:
    return RKPhi(order, tableau(tableau_name), cfl, nx)


def sequential(phi, u0: np.ndarray, nt: int) -> np.ndarray:
    """Sequential time stepping u^{n+1} = Phi u^n, u^0 = u0."""
    U = np.empty((nt + 1, u0.shape[-1]))
    U[0] = u0
    for n in range(nt):
        U[n + 1] = phi(U[n])
    return U


def dense_matrix(phi, nx: int) -> np.ndarray:
    """Dense matrix of a linear operator: column j = phi(e_j)."""
    return np.stack([phi(np.eye(nx)[j]) for j in range(nx)], axis=1)


# ---------------------------------------------------------------------------
# Stability function R(z) = 1 + z b^T (I - zA)^{-1} 1 (Lemma 1)
# ---------------------------------------------------------------------------
def stability_function(tab: Tableau, zc: np.ndarray) -> np.ndarray:
    """R(z): one stage-form step applied to the scalar test equation y' = lambda y,
    z = lambda dt (Lemma 1 proof: decouple into scalar ODEs).

    ERK:   k_i = z (1 + sum_{l<i} a_il k_l)
    SDIRK: k_i = z y_i,  y_i = (1 + sum_{l<i} a_il k_l) / (1 - a_ii z)
    R = 1 + sum_i b_i k_i."""
    zc = np.asarray(zc, dtype=complex)
    ks = []
    for i in range(tab.s):
        y = np.ones_like(zc)
        for l in range(i):
            y = y + tab.A[i][l] * ks[l]
        if tab.implicit:
            y = y / (1.0 - tab.A[i][i] * zc)
        ks.append(zc * y)
    out = np.ones_like(zc)
    for i in range(tab.s):
        out = out + tab.b[i] * ks[i]
    return out


def stencil_symbol(stencil: Dict[int, float], theta: np.ndarray) -> np.ndarray:
    """Eigenvalue of a circulant stencil on mode e^{i theta x}: sum_d a_d e^{i theta d}."""
    return sum(a * np.exp(1j * theta * d) for d, a in stencil.items())


def cfl_limit(order: int, tableau_name: str, ntheta: int = 20001, tol: float = 1e-12,
              excess: float = 0.0) -> float:
    """Largest c with max_theta |R(-c sigma_p(theta))| <= 1 + excess (Table 1).

    Bisection over c; |R| is evaluated on a theta grid.  `excess` is the
    tolerance on |R| <= 1 (R7)."""
    tab = tableau(tableau_name)
    theta = np.linspace(0.0, np.pi, ntheta)
    w, den = UPWIND[order]
    sig = stencil_symbol({d: float(wd) / float(den) for d, wd in w.items()}, theta)

    def stable(c):
        return np.max(np.abs(stability_function(tab, -c * sig))) <= 1.0 + excess

    lo, hi = 0.0, 4.0
    while hi - lo > tol:
        mid = 0.5 * (lo + hi)
        if stable(mid):
            lo = mid
        else:
            hi = mid
    return lo

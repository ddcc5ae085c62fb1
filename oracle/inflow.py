"""Oracle: inflow/outflow boundaries (§4.5).

ORACLE — test infrastructure only (see oracle/__init__.py).

The paper replaces the periodic boundary by an inflow u(-1, t) = g(t) at x = -1 and an
outflow at x = 1 and states only the ingredients of the closure:
"sufficiently accurate extrapolation is used at the outflow boundary; at the inflow
boundary, sufficiently accurate ERK stage values are computed using ideas similar to those
in Carpenter et al. ... we employ truncated Taylor series about the boundary and use the PDE
with the 'inverse Lax-Wendroff' procedure".  DESIGN.md reading R20 fixes the details:

* Grid: x_i = -1 + i dx, dx = 2/nx, i = 0..nx; x_0 = -1 is the inflow point (its value is
  data), the unknowns are u_1..u_nx (array index a = i - 1), x_nx = 1 is the outflow point.
* Inflow ghosts (array index a < 0, i.e. x_{-k} with k = -(a+1) >= 0): the exact solution
  near x = -1 is u(x, t) = g(t - (x + 1)/alpha), so the inverse Lax-Wendroff identity
  d^j u/dx^j = (-1/alpha)^j g^(j) turns the Taylor series about x_0 truncated after the
  p-th term into  u(x_{-k}, t) ~ sum_{j<=p} (k dx/alpha)^j / j! g^(j)(t).
  ERK stage values (Carpenter et al.): for du/dt = L u the stage vector of step n is
  Y_i = sum_q dt^q (A^q 1)_i d^q u/dt^q (t_n) (A strictly lower triangular, q < s), so the
  ghost value of stage i is  sum_{q<s} dt^q (A^q 1)_i sum_{j<=p} (k dx/alpha)^j/j! g^(q+j)(t_n).
* Outflow ghosts (a >= nx): polynomial extrapolation of degree p through the last p+1
  values of the vector the stencil acts on (each stage vector).
* Homogeneous part (error equations, coarse levels): inflow ghosts 0.
* Psi on an inflow/outflow grid: the periodic problem's LSQ Psi (same nx, c, m) truncated at
  the boundaries -- Toeplitz, no wrap (caption of tab:LSQlin_ERK_inflow P:685).

Phi is affine: Phi(u; t_n) = Phi_h u + b_n with b_n = Phi(0; t_n).  MGRIT runs on the
right-hand-side form U[n+1] = Phi_h U[n] + b_n (oracle.mgrit, R12) with the fine
right-hand side g_0 = (u0, b_0, ..., b_{nt-1}).
"""
from __future__ import annotations

import math
from fractions import Fraction
from typing import Dict, List, Optional

import numpy as np

from .discretization import Tableau, tableau, z_coefficients


def extrapolation_weights(p: int, k: int) -> List[Fraction]:
    """Lagrange weights e_j (j = 0..p) with u(N + k) = sum_j e_j u(N - j) exact for every
    polynomial of degree <= p (nodes N, N-1, ..., N-p, evaluated at N + k)."""
    out = []
    for j in range(p + 1):
        w = Fraction(1)
        for l in range(p + 1):
            if l != j:
                w *= Fraction(k + l, l - j)
        out.append(w)
    return out


def stage_powers(tab: Tableau) -> np.ndarray:
    """(A^q 1)_i for q = 0..s-1, i = 0..s-1 (row q)."""
    s = tab.s
    A = np.array(tab.A, dtype=float)
    v = np.ones(s)
    out = []
    for _ in range(s):
        out.append(v.copy())
        v = A @ v
    return np.array(out)


class BoundedRKPhi:
    """u -> Phi(u; t_n) for ERKp + Up on the inflow/outflow grid (stage form).

    `dg` is the row of inflow derivatives g^(r)(t_n), r = 0..p+s-1 (None: homogeneous,
    inflow ghosts 0)."""

    def __init__(self, order: int, tab_name: str, cfl: float, nx: int, alpha: float = 1.0):
        self.order, self.cfl, self.nx, self.alpha = order, cfl, nx, alpha
        self.tab = tableau(tab_name)
        assert not self.tab.implicit, "the paper's inflow/outflow runs are explicit (P:680)"
        self.z = z_coefficients(order, cfl)
        self.nl = -min(self.z)             # ghosts to the left
        self.nr = max(0, max(self.z))      # ghosts to the right
        self.dx = 2.0 / nx
        self.dt = cfl * self.dx / alpha
        self.ext = [[float(w) for w in extrapolation_weights(order, k)] for k in range(1, self.nr + 1)]
        self.apow = stage_powers(self.tab)
        self.nq = order + self.tab.s       # derivatives g^(0..p+s-1) needed

    def ghost_stage(self, i: int, dg: Optional[np.ndarray]) -> np.ndarray:
        """Inflow ghost values of stage i at x_{-k}, k = 0..nl-1 (R20)."""
        g = np.zeros(self.nl)
        if dg is None:
            return g
        for k in range(self.nl):
            acc = 0.0
            for q in range(self.tab.s):
                for j in range(self.order + 1):
                    acc += (self.dt ** q * self.apow[q][i]) * \
                        ((k * self.dx / self.alpha) ** j / math.factorial(j)) * dg[q + j]
            g[k] = acc
        return g

    def apply_z(self, y: np.ndarray, ghost_left: np.ndarray) -> np.ndarray:
        """(Z y)_a = sum_d z_d y~_{a+d}, y~ = y extended by the ghosts (d ascending)."""
        nx, p = self.nx, self.order
        ext = np.zeros(nx + self.nl + self.nr)
        ext[self.nl:self.nl + nx] = y
        for k in range(self.nl):                    # array index -(k+1) <-> x_{-k}
            ext[self.nl - 1 - k] = ghost_left[k]
        for kk in range(self.nr):                   # array index nx + kk <-> x_{nx+1+kk}
            ext[self.nl + nx + kk] = sum(w * y[nx - 1 - j] for j, w in enumerate(self.ext[kk]))
        out = None
        for d in sorted(self.z):
            term = self.z[d] * ext[self.nl + d:self.nl + d + nx]
            out = term if out is None else out + term
        return out

    def step(self, u: np.ndarray, dg: Optional[np.ndarray]) -> np.ndarray:
        A, b = self.tab.A, self.tab.b
        ks = []
        for i in range(self.tab.s):
            y = u
            for l in range(i):
                if A[i][l] != 0.0:
                    y = y + A[i][l] * ks[l]
            ks.append(self.apply_z(y, self.ghost_stage(i, dg)))
        out = u
        for i in range(self.tab.s):
            if b[i] != 0.0:
                out = out + b[i] * ks[i]
        return out

    def __call__(self, u: np.ndarray) -> np.ndarray:
        """Homogeneous part Phi_h (rows of a 2-D array are stepped independently)."""
        if u.ndim == 1:
            return self.step(u, None)
        return np.stack([self.step(r, None) for r in u])

    def forcing(self, dgs: np.ndarray) -> np.ndarray:
        """b_n = Phi(0; t_n) for every row dgs[n] (n = 0..nt-1)."""
        z = np.zeros(self.nx)
        return np.stack([self.step(z, dgs[n]) for n in range(dgs.shape[0])])


class TruncatedStencilPhi:
    """u -> Psi_T u, the stencil Psi truncated at the boundaries: (Psi_T u)_a =
    sum_{d: 0 <= a+d < nx} psi_d u_{a+d} (Toeplitz, no wrap)."""

    def __init__(self, stencil: Dict[int, float], nx: int):
        self.stencil = dict(sorted(stencil.items()))
        self.nx = nx
        self.nnz = len(stencil)

    def __call__(self, u):
        nx = self.nx
        out = np.zeros_like(u)
        first = True
        for d, c in self.stencil.items():
            term = np.zeros_like(u)
            lo, hi = max(0, -d), min(nx, nx - d)
            if hi > lo:
                term[..., lo:hi] = u[..., lo + d:hi + d]
            out = c * term if first else out + c * term
            first = False
        return out


def sequential(phi: BoundedRKPhi, u0: np.ndarray, dgs: np.ndarray) -> np.ndarray:
    """Sequential stepping U[n+1] = Phi(U[n]; t_n) (P:137-141 with boundary data)."""
    nt = dgs.shape[0]
    U = np.empty((nt + 1, phi.nx))
    U[0] = u0
    for n in range(nt):
        U[n + 1] = phi.step(U[n], dgs[n])
    return U


def fine_rhs(phi: BoundedRKPhi, u0: np.ndarray, dgs: np.ndarray) -> np.ndarray:
    """g_0 = (u0, b_0, ..., b_{nt-1}) of the fine level's RHS form (R12)."""
    g = np.empty((dgs.shape[0] + 1, phi.nx))
    g[0] = u0
    g[1:] = phi.forcing(dgs)
    return g

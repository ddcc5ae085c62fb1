"""Oracle: coarse-grid operators Psi (§2.2, §4).

ORACLE — test infrastructure only (see oracle/__init__.py).

* Psi_ideal = Phi^m.
* Rediscretised Psi: Phi rebuilt with time step m*dt, i.e. CFL m*c.
* Weighted linear least squares for the nonzeros psi of a sparse circulant
  Psi, eq. (LSQ_1D_problem), with w(z) = 1/(1-z+eps)^2, eps = 1e-6
  (P:338-342); solved as the complex least-squares problem, imaginary part
  truncated and flagged if larger than 1e-8.
* Sparsity patterns: a contiguous window centred on the characteristic
  departure point (R8), or thresholding of the ideal first
  column at eta*max.
* Multilevel: Psi_{l+1} ~ Phi_l^m recursively.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Dict, List, Sequence

import numpy as np

from .discretization import first_column


def ideal_first_column(phi: Callable, nx: int, m: int) -> np.ndarray:
    """First column of Phi^m: Phi applied m times to e_0."""
    e0 = np.zeros(nx)
    e0[0] = 1.0
    col = e0
    for _ in range(m):
        col = phi(col)
    return col


def eigenvalues(col: np.ndarray) -> np.ndarray:
    """Eigenvalues of a circulant = DFT of its first column."""
    return np.fft.fft(col)


def weights(lam: np.ndarray, eps: float = 1e-6) -> np.ndarray:
    """w_k = w(|lambda_k|) = 1/(1 - |lambda_k| + eps)^2."""
    return 1.0 / (1.0 - np.abs(lam) + eps) ** 2


def round_half_away(x: float) -> int:
    return int(math.floor(abs(x) + 0.5)) * (1 if x >= 0 else -1)


def window_pattern(shift: float, nu: int) -> List[int]:
    """nu contiguous offsets centred on the departure point -shift (R8)."""
    centre = round_half_away(-shift)
    h = (nu - 1) // 2
    return list(range(centre - h, centre - h + nu))


def threshold_pattern(col: np.ndarray, eta: float) -> List[int]:
    """Offsets d of entries with |(Phi^m)_{-d}| >= eta*max; contiguous hull."""
    nx = col.shape[0]
    thr = eta * np.max(np.abs(col))
    js = np.nonzero(np.abs(col) >= thr)[0]
    ds = sorted(((-j + nx // 2) % nx) - nx // 2 for j in js)   # d = -j wrapped to (-nx/2, nx/2]
    return list(range(ds[0], ds[-1] + 1))


@dataclass
class LSQResult:
    offsets: List[int]
    coeffs: np.ndarray
    imag_residue: float
    accepted: bool

    @property
    def stencil(self) -> Dict[int, float]:
        return {d: float(a) for d, a in zip(self.offsets, self.coeffs)}


def lsq_psi(target_col: np.ndarray, lam_fine: np.ndarray, offsets: Sequence[int],
            w: np.ndarray = None) -> LSQResult:
    """psi = argmin || W^{1/2} F (phi~^m - R^T psi) ||_2^2, eq. (LSQ_1D_problem) P:360-371.

    F is the DFT matrix (first-column convention P:359), R^T places psi_d at
    first-column index (-d mod nx).  Complex least squares; the real part is
    kept (Lemma 3) and results with |imag| > 1e-8 are flagged."""
    nx = target_col.shape[0]
    if w is None:
        w = weights(lam_fine)
    sw = np.sqrt(w)
    k = np.arange(nx)
    # column for offset d:  F e_{(-d) mod nx}  evaluated at frequency k
    cols = [np.exp(-2j * np.pi * k * ((-d) % nx) / nx) for d in offsets]
    A = sw[:, None] * np.stack(cols, axis=1)
    b = sw * np.fft.fft(target_col)
    sol, *_ = np.linalg.lstsq(A, b, rcond=None)
    imag = float(np.max(np.abs(sol.imag)))
    return LSQResult(list(offsets), sol.real.copy(), imag, imag <= 1e-8)


def redisc_cfl(cfl: float, m: int) -> float:
    """Coarse CFL of the rediscretised operator: time step m*dt."""
    return m * cfl


def fit_hierarchy(phi_fine: Callable, nx: int, m: int, cfl: float,
                  widths: Sequence[int] = (), eta: float = None) -> List[LSQResult]:
    """Psi_2..Psi_L by recursive weighted LSQ.

    Level l+1 approximates Phi_l^m with Phi_1 = phi_fine and Phi_l = Psi_l;
    the weights use |eigenvalues of Phi_l|.  Pattern: window of width
    widths[l] centred on -m^l c (R8), or the eta-threshold pattern (P:786,
    two-level only)."""
    out: List[LSQResult] = []
    phi = phi_fine
    nlev = len(widths) if eta is None else 1
    for lvl in range(nlev):
        e0 = np.zeros(nx)
        e0[0] = 1.0
        lam = eigenvalues(phi(e0))
        target = ideal_first_column(phi, nx, m)
        if eta is not None:
            offs = threshold_pattern(target, eta)
        else:
            offs = window_pattern(m ** (lvl + 1) * cfl, widths[lvl])
        res = lsq_psi(target, lam, offs)
        out.append(res)
        phi = _stencil_op(res.stencil)
    return out


def _stencil_op(stencil):
    from .discretization import apply_stencil

    def op(u):
        return apply_stencil(u, stencil)
    return op

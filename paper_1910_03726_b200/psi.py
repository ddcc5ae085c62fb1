"""Host-side synthesis of the coarse operators Psi (§4) — an INPUT of the library.

North star: "Psi's coefficients come from the paper's least-squares fit to its Fourier
error estimate, computed once on the host, and are an input to the library."

* eigenvalues of Phi from the stability function R(z) = 1 + z b^T (I - zA)^{-1} 1
  (Lemma 1) at the Fourier symbol of Z = dt L, with the library's own
  coefficients (`binding.scheme_coefficients`);
* weighted linear least squares eq. (LSQ_1D_problem) P:360-371 with
  w(z) = 1/(1-z+eps)^2, eps = 1e-6, solved as a *real* least-squares
  problem (Lemma 3 P:378-392 guarantees a real minimiser; the imaginary part the
  complex formulation would carry is what P:394 flags);
* patterns: contiguous window centred on -m^l c (R8) or eta_tol
  thresholding of the first column of Phi^m = IDFT(lambda^m);
* recursion Psi_{l+1} ~ Psi_l^m.
"""
from __future__ import annotations

import math
from typing import Dict, List, Sequence

import numpy as np

from . import binding


def stability_R(zc: np.ndarray, A: np.ndarray, b: np.ndarray) -> np.ndarray:
    """R(z) = 1 + z b^T (I - zA)^{-1} 1 for lower-triangular A (forward substitution)."""
    s = len(b)
    zc = np.asarray(zc, dtype=complex)
    x = []
    for i in range(s):
        acc = np.ones_like(zc)
        for j in range(i):
            acc = acc + zc * A[i, j] * x[j]
        x.append(acc / (1.0 - zc * A[i, i]))
    return 1.0 + zc * sum(b[i] * x[i] for i in range(s))


def symbol(stencil: Dict[int, float], nx: int) -> np.ndarray:
    theta = 2.0 * np.pi * np.arange(nx) / nx
    return sum(a * np.exp(1j * theta * d) for d, a in stencil.items())


def phi_eigenvalues(order: int, tableau: str, cfl: float, nx: int) -> np.ndarray:
    z, A, b = binding.scheme_coefficients(order, tableau, cfl)
    return stability_R(symbol(z, nx), A, b)


def window(shift: float, nu: int) -> List[int]:
    centre = int(math.floor(abs(shift) + 0.5)) * (-1 if shift > 0 else 1)
    lo = centre - (nu - 1) // 2
    return list(range(lo, lo + nu))


def threshold(lam_m: np.ndarray, eta: float) -> List[int]:
    col = np.real(np.fft.ifft(lam_m))           # first column of Phi^m
    nx = col.shape[0]
    keep = np.nonzero(np.abs(col) >= eta * np.abs(col).max())[0]
    ds = sorted(((-j + nx // 2) % nx) - nx // 2 for j in keep)
    return list(range(ds[0], ds[-1] + 1))


IMAG_TOL = 1e-8   # "if an imaginary component larger than 1e-8 is detected, we flag"


class PsiRejected(ValueError):
    """The LSQ solution was flagged and is not accepted as a coarse operator."""


def lsq(lam: np.ndarray, m: int, offsets: Sequence[int], eps: float = 1e-6,
        return_imag: bool = False):
    """Weighted LSQ  min || W^{1/2} (lambda^m - mu(psi)) ||  (eq. LSQ_1D_problem).

    Solved in the real form (Lemma 3, guarantees a real minimiser); the complex
    least-squares problem the paper solves is solved as well and its largest imaginary
    component is the P:394 flag (return_imag=True returns it)."""
    nx = lam.shape[0]
    theta = 2.0 * np.pi * np.arange(nx) / nx
    sw = 1.0 / (1.0 - np.abs(lam) + eps)
    M = sw[:, None] * np.exp(1j * np.outer(theta, np.asarray(offsets, dtype=float)))
    rhs = sw * lam ** m
    Ar = np.concatenate([M.real, M.imag], axis=0)
    br = np.concatenate([rhs.real, rhs.imag])
    psi, *_ = np.linalg.lstsq(Ar, br, rcond=None)
    if not return_imag:
        return psi
    pc, *_ = np.linalg.lstsq(M, rhs, rcond=None)
    return psi, float(np.max(np.abs(pc.imag)))


def hierarchy(order: int, tableau: str, cfl: float, nx: int, m: int, levels: int,
              widths: Sequence[int] = (), eta: float = None,
              allow_flagged: bool = False) -> List[Dict]:
    """Psi_2..Psi_L as library inputs [{"kind": "stencil", "offsets", "coeffs"}, ...].
    Each entry also carries the P:394 flag ("imag": largest imaginary component of the
    complex LSQ solution); a flagged fit (> 1e-8) raises PsiRejected unless allow_flagged."""
    lam = phi_eigenvalues(order, tableau, cfl, nx)
    out = []
    for lvl in range(levels - 1):
        if eta is not None:
            offs = threshold(lam ** m, eta)
        else:
            offs = window(m ** (lvl + 1) * cfl, widths[lvl])
        psi, imag = lsq(lam, m, offs, return_imag=True)
        if imag > IMAG_TOL and not allow_flagged:
            raise PsiRejected(f"level {lvl + 2}: LSQ imaginary component {imag:.2e} > 1e-8 "
                              f"(P:394) for offsets {offs[0]}..{offs[-1]}")
        out.append({"kind": "stencil", "offsets": offs, "coeffs": [float(c) for c in psi],
                    "imag": imag})
        lam = symbol(dict(zip(offs, psi)), nx)
    return out

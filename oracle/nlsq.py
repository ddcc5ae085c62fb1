"""Oracle: nonlinear least-squares coarse operators (Appendix B).

ORACLE — test infrastructure only (see oracle/__init__.py).

Problem (eq. (nlsq)): for a sparse circulant Psi with real nonzeros psi_a at the
offsets d_a (eigenvalues mu_k = sum_a psi_a e^{i theta_k d_a}),

    minimise  F(psi) = (1/nx) sum_k ||E_k(psi)||_2^2,

with ||E_k|| taken as the two-level FCF estimate (Dobrev_bounds) P:283-293,
    ||E_k|| = sqrt(m) |lam_k|^m |lam_k^m - mu_k| / (1 - |mu_k|) (1 - |mu_k|^(nt/m - 1)).
The trailing quotient is the finite geometric sum g(a) = sum_{j=0}^{N-2} a^j, a = |mu_k|,
N = nt/m, which is how it is evaluated here (Horner): defined for every a, including the
consistent mode a = 1 where the closed form is 0/0.

Reading (R21; the paper says only "MATLAB's lsqnonlin ... Levenberg-Marquardt ...
default settings ... a maximum of 30 nonlinear iterations", started from the linear LSQ
solution):
* residuals: the complex numbers r_k = C_k g(|mu_k|) (lam_k^m - mu_k), C_k = sqrt(m) |lam_k|^m,
  as 2 nx real residuals (|r_k| = ||E_k||, so F is the paper's objective, and r is smooth
  where lam_k^m = mu_k);
* Levenberg-Marquardt with identity scaling: (J^T J + l I) delta = -J^T r, l_0 = 0.01, a step
  that lowers F is accepted and l <- l/10, otherwise l <- 10 l; every trial counts as an
  iteration (at most max_iter = 30); stop after an accepted step with F_old - F_new <=
  1e-6 F_old or ||delta|| <= 1e-6 (1 + ||psi||).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

import numpy as np


def geometric_sum(a: np.ndarray, n_terms: int):
    """g(a) = sum_{j=0}^{n_terms-1} a^j and g'(a), by Horner (n_terms >= 1)."""
    g = np.ones_like(a)
    dg = np.zeros_like(a)
    for _ in range(n_terms - 1):
        dg = dg * a + g
        g = g * a + 1.0
    return g, dg


def symbol(psi: np.ndarray, offsets: Sequence[int], nx: int) -> np.ndarray:
    """mu_k = sum_a psi_a e^{i theta_k d_a}, theta_k = 2 pi k/nx."""
    k = np.arange(nx)
    mu = np.zeros(nx, dtype=complex)
    for p, d in zip(psi, offsets):
        mu = mu + p * np.exp(2j * np.pi * ((k * d) % nx) / nx)
    return mu


def residuals(psi: np.ndarray, offsets: Sequence[int], lam: np.ndarray, m: int, nt: int) -> np.ndarray:
    """r_k = sqrt(m) |lam_k|^m g(|mu_k|) (lam_k^m - mu_k)  (complex; |r_k| = (Dobrev_bounds))."""
    nx = lam.shape[0]
    mu = symbol(psi, offsets, nx)
    g, _ = geometric_sum(np.abs(mu), nt // m - 1)
    return np.sqrt(m) * np.abs(lam) ** m * g * (lam ** m - mu)


def objective(psi, offsets, lam, m, nt) -> float:
    """F(psi) = (1/nx) sum_k |r_k|^2, eq. (nlsq) P:1052-1061."""
    r = residuals(psi, offsets, lam, m, nt)
    return float(np.sum(np.abs(r) ** 2) / lam.shape[0])


def jacobian(psi, offsets, lam, m, nt) -> np.ndarray:
    """dr_k/dpsi_a (complex nx x nu): C [g'(a) da/dpsi_a (lam^m - mu) - g(a) E_a],
    E_a = e^{i theta_k d_a}, da/dpsi_a = Re(conj(mu) E_a)/a."""
    nx = lam.shape[0]
    k = np.arange(nx)
    mu = symbol(psi, offsets, nx)
    a = np.abs(mu)
    g, dg = geometric_sum(a, nt // m - 1)
    C = np.sqrt(m) * np.abs(lam) ** m
    delta = lam ** m - mu
    J = np.empty((nx, len(offsets)), dtype=complex)
    for col, d in enumerate(offsets):
        E = np.exp(2j * np.pi * ((k * d) % nx) / nx)
        da = np.where(a > 0, np.real(np.conj(mu) * E) / np.where(a > 0, a, 1.0), 0.0)
        J[:, col] = C * (dg * da * delta - g * E)
    return J


@dataclass
class NLSQResult:
    offsets: List[int]
    coeffs: np.ndarray
    objective: float
    history: List[float]      # F after every iteration (trial), history[0] = F(psi_0)
    accepted: List[bool]
    iterations: int

    @property
    def stencil(self):
        return {d: float(c) for d, c in zip(self.offsets, self.coeffs)}


def nlsq_psi(psi0: np.ndarray, offsets: Sequence[int], lam: np.ndarray, m: int, nt: int,
             max_iter: int = 30) -> NLSQResult:
    """Levenberg-Marquardt on eq. (nlsq) from psi0 (the linear LSQ solution); R21."""
    nx = lam.shape[0]
    psi = np.array(psi0, dtype=float)
    nu = psi.shape[0]
    lmb = 0.01
    F = objective(psi, offsets, lam, m, nt)
    hist, acc = [F], []
    it = 0
    while it < max_iter:
        r = residuals(psi, offsets, lam, m, nt)
        J = jacobian(psi, offsets, lam, m, nt)
        Jr = np.vstack([J.real, J.imag])                 # 2 nx real residuals
        rr = np.concatenate([r.real, r.imag])
        done = False
        while it < max_iter:
            it += 1
            # (J^T J + l I) delta = -J^T r as the augmented least-squares problem
            A = np.vstack([Jr, np.sqrt(lmb) * np.eye(nu)])
            b = np.concatenate([-rr, np.zeros(nu)])
            delta, *_ = np.linalg.lstsq(A, b, rcond=None)
            Fn = objective(psi + delta, offsets, lam, m, nt)
            if Fn < F:
                small = (F - Fn) <= 1e-6 * F or np.linalg.norm(delta) <= 1e-6 * (1.0 + np.linalg.norm(psi))
                psi = psi + delta
                F = Fn
                lmb /= 10.0
                hist.append(F)
                acc.append(True)
                done = small
                break
            lmb *= 10.0
            hist.append(Fn)
            acc.append(False)
        if done:
            break
    return NLSQResult(list(offsets), psi, F, hist, acc, it)

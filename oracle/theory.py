"""Oracle: two-level convergence theory (§3.1).

ORACLE — test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np


def fcf_bound(lam: np.ndarray, mu: np.ndarray, m: int, nt: int) -> np.ndarray:
    """||E_k||_2 <= sqrt(m) |lam|^m |lam^m - mu| / (1 - |mu|) (1 - |mu|^(nt/m - 1)),
    eq. (Dobrev_bounds) P:283-293 (valid for |lam|, |mu| < 1)."""
    lam = np.asarray(lam, dtype=complex)
    mu = np.asarray(mu, dtype=complex)
    amu = np.abs(mu)
    return (np.sqrt(m) * np.abs(lam) ** m * np.abs(lam ** m - mu) / (1.0 - amu)
            * (1.0 - amu ** (nt // m - 1)))


def scalar_two_level_error_matrix(lam: complex, mu: complex, m: int, nt: int,
                                  relax: str = "FCF") -> np.ndarray:
    """Dense error-propagation matrix of one two-level iteration for the scalar
    problem u^{n+1} = lam u^n with coarse stepper mu, built column
    by column by running the iteration on unit errors (e^0 pinned to zero)."""
    cols = []
    for n0 in range(1, nt + 1):
        e = np.zeros(nt + 1, dtype=complex)
        e[n0] = 1.0
        cols.append(_scalar_iteration(e, lam, mu, m, relax))
    return np.stack(cols, axis=1)[1:, :]


def _scalar_iteration(e, lam, mu, m, relax):
    e = e.copy()
    nt = len(e) - 1

    def frelax():
        for j in range(0, nt, m):
            for i in range(1, m):
                e[j + i] = lam * e[j + i - 1]

    def crelax():
        for j in range(m, nt + 1, m):
            e[j] = lam * e[j - 1]

    frelax()
    if relax == "FCF":
        crelax()
        frelax()
    nc = nt // m
    r = np.zeros(nc + 1, dtype=complex)
    for j in range(1, nc + 1):
        r[j] = lam * e[j * m - 1] - e[j * m]
    ec = np.zeros(nc + 1, dtype=complex)
    for j in range(1, nc + 1):
        ec[j] = mu * ec[j - 1] + r[j]
    for j in range(1, nc + 1):
        e[j * m] = e[j * m] + ec[j]
    frelax()
    return e

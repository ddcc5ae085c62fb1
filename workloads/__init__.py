"""Seeded synthetic inputs shared by the oracle and the product path.

This module holds NO arithmetic of the method (no stencils, no Runge-Kutta,
no MGRIT, no Psi fitting).  It only states the five BASELINE.json workloads as
plain parameters and generates their inputs:

* the initial condition u0 (PAPER.md P:73 for sin^4(pi x); BASELINE.json
  configs 2-5 for the random Fourier modes and the Gaussian, read per
  DESIGN.md reading R11),
* the random initial space-time iterate ("uniformly random except at t = 0",
  PAPER.md P:218), produced by a counter-based generator so that any row can
  be regenerated on its own (and so that the CUDA library can implement the
  very same integer generator on the device, reading R4).

Both `oracle/` and `paper_1910_03726_b200/` import it; neither imports the
other.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np

# ----------------------------------------------------------------------------
# Counter-based uniform generator (SplitMix64 finaliser).
#   key(seed, idx) = idx + seed * GOLDEN2   (mod 2^64)
#   z = splitmix64(key);  k = z >> 11  (53 random bits)
#   U[-1,1):  (k - 2^52) * 2^-52   (exact in fp64)
#   U[0, 1):   k * 2^-53           (exact in fp64)
# idx = n * nx + i for space-time point (n, i).
# ----------------------------------------------------------------------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
GOLDEN2 = np.uint64(0x632BE59BD9B4E019)
MIX1 = np.uint64(0xBF58476D1CE4E5B9)
MIX2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * MIX1
        z = (z ^ (z >> np.uint64(27))) * MIX2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_from_index(seed: int, idx: np.ndarray, lo: float) -> np.ndarray:
    """Uniform variates for flat indices `idx`; lo = -1.0 -> U[-1,1), lo = 0.0 -> U[0,1)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = idx + np.uint64(seed) * GOLDEN2
    k = (splitmix64(key) >> np.uint64(11)).astype(np.int64)
    if lo == -1.0:
        return (k - (1 << 52)).astype(np.float64) * 2.0 ** -52
    if lo == 0.0:
        return k.astype(np.float64) * 2.0 ** -53
    raise ValueError("lo must be -1.0 or 0.0")


def guess_rows(seed: int, nx: int, rows: np.ndarray, lo: float = -1.0) -> np.ndarray:
    """Rows `rows` of the random initial iterate, shape (len(rows), nx).

    Row 0 of the iterate is replaced by u0 by the caller (`initial_iterate`)."""
    rows = np.asarray(rows, dtype=np.int64).reshape(-1)
    idx = (rows[:, None].astype(np.uint64) * np.uint64(nx)
           + np.arange(nx, dtype=np.uint64)[None, :])
    return uniform_from_index(seed, idx, lo)


def initial_iterate(seed: int, nx: int, nt: int, u0: np.ndarray, lo: float = -1.0) -> np.ndarray:
    """Full (nt+1) x nx initial space-time iterate, row 0 = u0."""
    U = np.empty((nt + 1, nx), dtype=np.float64)
    chunk = max(1, (1 << 22) // nx)
    for r0 in range(0, nt + 1, chunk):
        r1 = min(nt + 1, r0 + chunk)
        U[r0:r1] = guess_rows(seed, nx, np.arange(r0, r1), lo)
    U[0] = u0
    return U


# ----------------------------------------------------------------------------
# Grid and initial conditions.  x_i = -1 + i*dx, dx = 2/nx, periodic (R17).
# ----------------------------------------------------------------------------
def grid(nx: int) -> np.ndarray:
    return -1.0 + np.arange(nx, dtype=np.float64) * (2.0 / nx)


def u0_sin4(nx: int) -> np.ndarray:
    """u(x,0) = sin^4(pi x)."""
    return np.sin(np.pi * grid(nx)) ** 4


def u0_fourier(nx: int, seed: int, modes: int = 8) -> np.ndarray:
    """Random smooth sum of `modes` Fourier modes, a_k, b_k ~ N(0, 1/k^2) (BJ cfg2; R11)."""
    rng = np.random.default_rng(seed)
    x = grid(nx)
    u = np.zeros(nx)
    for k in range(1, modes + 1):
        a, b = rng.normal(0.0, 1.0 / k, 2)
        u += a * np.cos(k * np.pi * x) + b * np.sin(k * np.pi * x)
    return u


def u0_gauss(nx: int) -> np.ndarray:
    """exp(-50 x^2) sampled on the periodic grid (BJ cfg3; wrap jump ~2e-22, R11)."""
    x = grid(nx)
    return np.exp(-50.0 * x * x)


# ----------------------------------------------------------------------------
# The BASELINE.json workloads, as plain parameters.
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class Workload:
    name: str
    nx: int
    nt: int
    cfl: float
    family: str            # "ERK" | "SDIRK"
    order: int             # p of ERKp/SDIRKp and of the U_p stencil
    tableau: str           # tableau id, e.g. "erk3_kutta", "erk3_ssp", "sdirk3"
    m: int
    levels: int
    relax: str             # "F" | "FCF"
    psi_kind: str          # "stencil" | "ideal" | "redisc"
    psi_widths: Tuple[int, ...] = ()   # nu per coarse level (stencil kind)
    psi_eta: Optional[float] = None    # threshold pattern instead of a window
    redisc_cfl: Optional[float] = None
    u0_kind: str = "sin4"
    u0_seed: int = 0
    guess_seed: int = 0
    guess_lo: float = -1.0
    tol: float = 1e-10
    max_iter: int = 128
    alpha: float = 1.0
    boundary: str = "periodic"   # "inflow": inflow u(-1,t) = sin^4(pi t) / outflow (PAPER.md 4.5)

    @property
    def dx(self) -> float:
        return 2.0 / self.nx

    @property
    def dt(self) -> float:
        return self.cfl * self.dx / self.alpha

    def u0(self) -> np.ndarray:
        if self.u0_kind == "sin4":
            return u0_sin4(self.nx)
        if self.u0_kind == "fourier":
            return u0_fourier(self.nx, self.u0_seed)
        if self.u0_kind == "gauss":
            return u0_gauss(self.nx)
        if self.u0_kind == "sin4_inflow":   # sin^4(pi x) on the unknowns x_1..x_nx
            return np.sin(np.pi * inflow_grid(self.nx)) ** 4
        raise ValueError(self.u0_kind)

    def guess(self) -> np.ndarray:
        return initial_iterate(self.guess_seed, self.nx, self.nt, self.u0(), self.guess_lo)

    def scaled(self, nx: int, nt: int, **kw) -> "Workload":
        """Same workload recipe on a smaller grid (parity-test sizes)."""
        d = dict(self.__dict__)
        d.update(nx=nx, nt=nt, name=f"{self.name}@{nx}x{nt}")
        d.update(kw)
        return Workload(**d)


CFG1_REDISC = Workload("cfg1_redisc", 64, 256, 0.85, "ERK", 1, "erk1", 2, 2, "F", "redisc",
                       redisc_cfl=1.7, u0_kind="sin4", guess_seed=0, max_iter=128)
CFG1_IDEAL = Workload("cfg1_ideal", 64, 256, 0.85, "ERK", 1, "erk1", 2, 2, "F", "ideal",
                      u0_kind="sin4", guess_seed=0, max_iter=128)
CFG2 = Workload("cfg2", 1024, 4096, 0.85, "ERK", 3, "erk3_kutta", 4, 2, "FCF", "stencil",
                psi_widths=(9,), u0_kind="fourier", u0_seed=1, guess_seed=2, max_iter=64)
CFG3 = Workload("cfg3", 4096, 16384, 0.85, "ERK", 5, "erk5", 8, 2, "FCF", "stencil",
                psi_widths=(15,), u0_kind="gauss", guess_seed=3, max_iter=64)
CFG4_LITERAL = Workload("cfg4_literal", 4096, 16384, 4.0, "SDIRK", 3, "sdirk3", 4, 2, "FCF",
                        "stencil", psi_widths=(11,), u0_kind="fourier", u0_seed=4,
                        guess_seed=5, max_iter=64)
CFG4 = Workload("cfg4", 4096, 16384, 4.0, "SDIRK", 3, "sdirk3", 4, 2, "FCF", "stencil",
                psi_eta=0.01, u0_kind="fourier", u0_seed=4, guess_seed=5, max_iter=64)
CFG5 = Workload("cfg5", 16384, 65536, 0.85, "ERK", 3, "erk3_ssp", 4, 6, "FCF", "stencil",
                psi_widths=(9, 13, 17, 21, 25), u0_kind="fourier", u0_seed=6, guess_seed=7,
                max_iter=64)

# Inflow/outflow runs shaped like tab:LSQlin_ERK_inflow: ERKp+Up, 2^12 x 2^14
# two-level m = 4 and a 2^10 x 2^12 four-level V-cycle, the periodic problem's LSQ Psi truncated
# at the boundaries (widths as for the periodic configs, R8).  Not BASELINE.json configs:
# measurement cases of SURVEY 8(f) NEXT-4.
INFLOW_ERK3 = Workload("inflow_erk3", 4096, 16384, 0.85, "ERK", 3, "erk3_ssp", 4, 2, "FCF", "stencil",
                       psi_widths=(9,), u0_kind="sin4_inflow", guess_seed=8, boundary="inflow")
INFLOW_ERK3_ML = Workload("inflow_erk3_ml", 1024, 4096, 0.85, "ERK", 3, "erk3_ssp", 4, 4, "FCF",
                          "stencil", psi_widths=(9, 13, 17), u0_kind="sin4_inflow", guess_seed=9,
                          boundary="inflow")

ALL = {w.name: w for w in (CFG1_REDISC, CFG1_IDEAL, CFG2, CFG3, CFG4_LITERAL, CFG4, CFG5,
                           INFLOW_ERK3, INFLOW_ERK3_ML)}


# ----------------------------------------------------------------------------
# Inflow data of the inflow/outflow problem (§4.5): u(-1, t) = sin^4(pi t).
# The derivative table g^(r)(t_n), r = 0..nq-1, is the boundary DATA both the oracle and the
# library consume; the inverse Lax-Wendroff / stage-value arithmetic that turns it into
# ghost values is the method's and lives on each side separately (R20).
# sin^4(y) = 3/8 - cos(2y)/2 + cos(4y)/8.
# ----------------------------------------------------------------------------
def inflow_sin4_derivatives(t: np.ndarray, nq: int) -> np.ndarray:
    """Rows n: g^(r)(t_n) for r = 0..nq-1, g(t) = sin^4(pi t)."""
    t = np.asarray(t, dtype=np.float64).reshape(-1)
    out = np.empty((t.shape[0], nq))
    for r in range(nq):
        ph = r * np.pi / 2.0
        v = -0.5 * (2.0 * np.pi) ** r * np.cos(2.0 * np.pi * t + ph) + \
            0.125 * (4.0 * np.pi) ** r * np.cos(4.0 * np.pi * t + ph)
        out[:, r] = v + (0.375 if r == 0 else 0.0)
    return out


def inflow_grid(nx: int) -> np.ndarray:
    """Unknowns of the inflow/outflow grid: x_i = -1 + i dx, i = 1..nx (x_0 = -1 is data)."""
    return -1.0 + np.arange(1, nx + 1, dtype=np.float64) * (2.0 / nx)

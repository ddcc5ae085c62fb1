"""Pins of the inflow/outflow oracle (oracle/inflow.py; §4.5, R20).

Each test names what fixes the result independently of the oracle's own formulas:
polynomial exactness (U_p, ERK_p and degree-p extrapolation are exact on polynomials of
degree <= p, so with consistent ghost stage values sequential stepping reproduces the exact
solution g(t - x - 1) to rounding), the convergence order p against the exact solution of
P:676's inflow, the Toeplitz structure away from the boundaries, the paper's iteration counts
of tab:LSQlin_ERK_inflow, and the MGRIT identities (ideal Psi, finite termination).
"""
import math
from fractions import Fraction

import numpy as np
import pytest
from numpy.polynomial import polynomial as Pl

import workloads as W
from oracle import discretization as D
from oracle import inflow as I
from oracle import mgrit as M
from oracle import psi as P

SCHEMES = [(1, "erk1", 0.85), (3, "erk3_ssp", 1.3), (3, "erk3_kutta", 1.3), (5, "erk5", 1.6)]


def _poly_derivs(coef, t, nq):
    out = np.zeros((len(t), nq))
    cc = np.array(coef, dtype=float)
    for r in range(nq):
        out[:, r] = Pl.polyval(t, cc)
        cc = Pl.polyder(cc) if len(cc) > 1 else np.zeros(1)
    return out


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("k", [1, 2])
def test_extrapolation_weights_exact_on_polynomials(p, k):
    """Lagrange extrapolation of degree p reproduces x^q, q <= p, exactly (and not x^(p+1))."""
    w = I.extrapolation_weights(p, k)
    for q in range(p + 2):
        val = sum(wj * Fraction(-j) ** q for j, wj in enumerate(w))
        if q <= p:
            assert val == Fraction(k) ** q
        else:
            assert val != Fraction(k) ** q
    if p == 3 and k == 1:
        assert w == [4, -6, 4, -1]


@pytest.mark.parametrize("order,tab,c", SCHEMES)
def test_polynomial_inflow_is_reproduced_exactly(order, tab, c):
    """With g a polynomial of degree <= p the exact solution u = g(t - x - 1) is a polynomial
    of degree <= p in x and t.  U_p differentiates it exactly, ERK_p integrates it exactly
    (R(z) = e^z up to z^p, L nilpotent on the space), the inverse Lax-Wendroff Taylor ghosts
    truncated after j = p and the degree-p outflow extrapolation are exact: so sequential
    stepping must reproduce it to rounding -- any error in the stage-value formula, a sign of
    the Taylor terms, the ghost indexing or the extrapolation weights breaks this."""
    nx, nt = 32, 40
    ph = I.BoundedRKPhi(order, tab, c, nx)
    rng = np.random.default_rng(order)
    coef = rng.normal(size=order + 1)
    t = np.arange(nt) * ph.dt
    x = W.inflow_grid(nx)
    U = I.sequential(ph, Pl.polyval(-(x + 1), coef), _poly_derivs(coef, t, ph.nq))
    ex = np.stack([Pl.polyval(n * ph.dt - (x + 1), coef) for n in range(nt + 1)])
    assert np.max(np.abs(U - ex)) / np.max(np.abs(ex)) < 5e-14


def test_naive_stage_boundary_values_are_not_exact():
    """Control for the pin above: ghost stage values g(t_n + c_i dt) (the classical boundary
    treatment that loses order, Carpenter et al.) are not exact for ERK3 on a cubic."""
    nx, nt = 32, 40
    ph = I.BoundedRKPhi(3, "erk3_ssp", 1.3, nx)
    coef = np.random.default_rng(3).normal(size=4)
    cs = ph.tab.c

    class Naive(I.BoundedRKPhi):
        def ghost_stage(self, i, dg):
            if dg is None:
                return np.zeros(self.nl)
            g = np.zeros(self.nl)
            for k in range(self.nl):   # g(t_n + c_i dt + k dx) by its Taylor series
                h = cs[i] * self.dt + k * self.dx
                g[k] = sum(h ** r / math.factorial(r) * dg[r] for r in range(self.nq))
            return g

    nv = Naive(3, "erk3_ssp", 1.3, nx)
    t = np.arange(nt) * ph.dt
    x = W.inflow_grid(nx)
    dg = _poly_derivs(coef, t, ph.nq)
    ex = np.stack([Pl.polyval(n * ph.dt - (x + 1), coef) for n in range(nt + 1)])
    err = np.max(np.abs(I.sequential(nv, Pl.polyval(-(x + 1), coef), dg) - ex))
    assert err > 1e-8


@pytest.mark.parametrize("order,tab,cmax", [(1, "erk1", 1.0), (3, "erk3_ssp", 1.625891),
                                            (5, "erk5", 1.96583)])
def test_convergence_order_against_exact_inflow_solution(order, tab, cmax):
    """inflow sin^4(pi t) at x = -1 with u0 = sin^4(pi x) has the exact solution
    sin^4(pi (x - t)); 'numerical tests ... verify that convergence at the theoretically
    predicted rates is achieved': error ratio ~ 2^p per halving of dx at c = 0.85 c_max."""
    c = 0.85 * cmax
    errs = []
    for nx in (64, 128, 256):
        ph = I.BoundedRKPhi(order, tab, c, nx)
        nt = int(round(1.0 / ph.dt))
        dgs = W.inflow_sin4_derivatives(np.arange(nt) * ph.dt, ph.nq)
        x = W.inflow_grid(nx)
        U = I.sequential(ph, np.sin(np.pi * x) ** 4, dgs)
        errs.append(np.max(np.abs(U[-1] - np.sin(np.pi * (x - nt * ph.dt)) ** 4)))
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(order - 0.2 < r < order + 0.4 for r in rates), rates


@pytest.mark.parametrize("order,tab,c", SCHEMES)
def test_interior_rows_equal_periodic_operator(order, tab, c):
    """Away from the boundaries the inflow/outflow Phi_h shares the periodic Phi's Toeplitz
    rows ('the same Toeplitz structure away from the boundaries')."""
    nx = 48
    ph = I.BoundedRKPhi(order, tab, c, nx)
    per = D.make_phi(order, tab, c, nx)
    A = np.stack([ph(np.eye(nx)[j]) for j in range(nx)], axis=1)
    B = np.stack([per(np.eye(nx)[j]) for j in range(nx)], axis=1)
    s = ph.tab.s
    lo, hi = s * ph.nl, nx - s * ph.nr
    np.testing.assert_allclose(A[lo:hi], B[lo:hi], atol=1e-15, rtol=0)
    assert not np.allclose(A[:lo], B[:lo])


def test_homogeneous_operator_is_stable_and_outflowing():
    """With zero inflow every error leaves the domain: ||Phi_h^n|| -> 0 (spectral radius < 1)."""
    for order, tab, cmax in [(1, "erk1", 1.0), (3, "erk3_ssp", 1.625891), (5, "erk5", 1.96583)]:
        ph = I.BoundedRKPhi(order, tab, 0.85 * cmax, 32)
        A = np.stack([ph(np.eye(32)[j]) for j in range(32)], axis=1)
        assert np.max(np.abs(np.linalg.eigvals(A))) < 1.0
        assert np.linalg.norm(np.linalg.matrix_power(A, 4 * 32), 2) < 1e-10


def test_erk1_u1_cfl1_is_exact_shift_with_inflow():
    """U1 + forward Euler at CFL 1: u_i^{n+1} = u_{i-1}^n and the first unknown receives the
    boundary value g(t_n) (P:406 on the inflow grid)."""
    nx, nt = 64, 20
    ph = I.BoundedRKPhi(1, "erk1", 1.0, nx)
    u = W.guess_rows(11, nx, np.array([3]))[0]
    dgs = W.inflow_sin4_derivatives(np.arange(nt) * ph.dt, ph.nq)
    U = I.sequential(ph, u, dgs)
    for n in range(nt):
        np.testing.assert_allclose(U[n + 1][1:], U[n][:-1], rtol=0, atol=2e-16)
        assert abs(U[n + 1][0] - dgs[n, 0]) <= 2e-16


def test_truncated_psi_is_toeplitz_without_wrap():
    """Psi_T: entries (a, a+d) = psi_d inside the grid, nothing wraps; the
    paper's characteristic patterns (offsets <= 0) make it lower triangular."""
    nx = 20
    st = {-4: 0.1, -3: 0.5, -2: 0.3, -1: 0.1}
    T = np.stack([I.TruncatedStencilPhi(st, nx)(np.eye(nx)[j]) for j in range(nx)], axis=1)
    ref = np.zeros((nx, nx))
    for a in range(nx):
        for d, v in st.items():
            if 0 <= a + d < nx:
                ref[a, a + d] = v
    assert np.array_equal(T, ref)
    assert np.array_equal(T, np.tril(T, -1))


def _inflow_solve(order, tab, c, nx, nt, m, ops_psi, relax="FCF", max_iter=60, seed=0):
    ph = I.BoundedRKPhi(order, tab, c, nx)
    dgs = W.inflow_sin4_derivatives(np.arange(nt) * ph.dt, ph.nq)
    x = W.inflow_grid(nx)
    u0 = np.sin(np.pi * x) ** 4
    g0 = I.fine_rhs(ph, u0, dgs)
    U = W.initial_iterate(seed, nx, nt, u0, 0.0)
    ops = [ph] + ops_psi(ph)
    rep = M.solve(U, ops, m, 2.0 / nx, ph.dt, relax, 1e-10, max_iter, g0=g0)
    return rep, U, ph, g0


@pytest.mark.parametrize("m,nu,kref", [(2, 2, 10), (4, 3, 6), (8, 4, 6)])
def test_paper_inflow_iteration_table(m, nu, kref):
    """tab:LSQlin_ERK_inflow, ERK1+U1, 2^8 x 2^10, two-level, m = 2, 4, 8:
    10, 6, 6 iterations with the periodic problem's LSQ Psi truncated at the boundaries
    (the same windows that reproduce the periodic tab:LSQlin_ERK, R8; U[0,1) guess R3;
    +-1 allowed for the unknown RNG stream, R16)."""
    nx, nt = 256, 1024
    per = D.make_phi(1, "erk1", 0.85, nx)
    fit = P.fit_hierarchy(per, nx, m, 0.85, (nu,))[0]
    rep, *_ = _inflow_solve(1, "erk1", 0.85, nx, nt, m,
                            lambda ph: [I.TruncatedStencilPhi(fit.stencil, nx)])
    assert rep.converged
    assert abs(rep.iterations - kref) <= 1, (rep.iterations, kref)


@pytest.mark.parametrize("order,tab,c,m", [(1, "erk1", 0.85, 2), (3, "erk3_ssp", 1.3, 4),
                                          (5, "erk5", 1.6, 4)])
def test_ideal_psi_one_iteration_with_inflow(order, tab, c, m):
    """Psi = Phi_h^m solves the inflow problem in one iteration."""
    rep, *_ = _inflow_solve(order, tab, c, 32, 64, m, lambda ph: [D.PowerPhi(ph, m)])
    assert rep.iterations == 1 and rep.converged


@pytest.mark.parametrize("relax,iters", [("FCF", 4), ("F", 8)])
def test_finite_termination_equals_sequential_rhs_form(relax, iters):
    """After nt/(2m) FCF (nt/m F) iterations the iterate is sequential stepping of the same
    affine system U[n+1] = Phi_h U[n] + b_n -- exact in exact arithmetic, in
    fp64 up to the rounding of the corrections -- and not one iteration earlier."""
    nx, nt, m = 32, 32, 4
    per = D.make_phi(3, "erk3_ssp", 1.3, nx)
    fit = P.fit_hierarchy(per, nx, m, 1.3, (9,))[0]
    psi = lambda ph: [I.TruncatedStencilPhi(fit.stencil, nx)]
    _, Ub, ph, g0 = _inflow_solve(3, "erk3_ssp", 1.3, nx, nt, m, psi, relax, iters - 1)
    ref = M.sequential_rhs(ph, g0)
    assert np.max(np.abs(Ub - ref)) > 1e-9
    rep, U, ph, g0 = _inflow_solve(3, "erk3_ssp", 1.3, nx, nt, m, psi, relax, iters)
    assert np.max(np.abs(U - ref)) < 1e-13 * np.max(np.abs(ref))
    # the fixed point is the boundary-forced sequential solution (up to rounding)
    seq = I.sequential(ph, g0[0], W.inflow_sin4_derivatives(np.arange(nt) * ph.dt, ph.nq))
    np.testing.assert_allclose(ref, seq, atol=1e-14, rtol=0)


def test_multilevel_inflow_converges_like_periodic():
    """V-cycles (m = 4) with the periodic Psi hierarchy truncated at the boundaries
    converge in a handful of iterations (tab:LSQlin_ERK_inflow right half, ERK1+U1 2^8 x 2^10:
    6 for 2..5 levels; the per-level patterns are figure-only, so +-1 around 7 here)."""
    nx, nt, m = 256, 1024, 4
    per = D.make_phi(1, "erk1", 0.85, nx)
    fits = P.fit_hierarchy(per, nx, m, 0.85, (3, 5, 7))   # widths: R8-style, unpinned
    rep, *_ = _inflow_solve(1, "erk1", 0.85, nx, nt, m,
                            lambda ph: [I.TruncatedStencilPhi(f.stencil, nx) for f in fits])
    assert rep.converged and rep.iterations <= 8, rep.iterations

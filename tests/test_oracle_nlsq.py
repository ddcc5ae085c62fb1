"""Pins of the nonlinear least-squares oracle (oracle/nlsq.py; Appendix B, P:1030-1068,
DESIGN.md R21).  What fixes the results independently of the oracle's own formulas: the closed
form of the geometric sum, the FCF estimate (Dobrev_bounds) as written in oracle/theory.py from
P:283-293, finite differences for the Jacobian, scipy's MINPACK Levenberg-Marquardt on the same
residuals, and the paper's iteration counts of tab:LSQnonlin_ERK."""
import numpy as np
import pytest

import workloads as W
from oracle import discretization as D
from oracle import mgrit as M
from oracle import nlsq as N
from oracle import psi as P
from oracle import theory as T


def _setup(order, tab, c, nx, m, nu):
    phi = D.make_phi(order, tab, c, nx)
    fit = P.fit_hierarchy(phi, nx, m, c, (nu,))[0]
    e0 = np.zeros(nx)
    e0[0] = 1.0
    lam = P.eigenvalues(phi(e0))
    return phi, fit, lam


def test_geometric_sum_closed_form_and_limit():
    a = np.array([0.0, 0.3, 0.9, 0.999, 1.0, 1.01])
    for n in (1, 2, 7, 200):
        g, dg = N.geometric_sum(a, n)
        for ai, gi, di in zip(a, g, dg):
            ref = n if ai == 1.0 else (1.0 - ai ** n) / (1.0 - ai)
            assert abs(gi - ref) <= 1e-11 * abs(ref)
            dref = sum(j * ai ** (j - 1) for j in range(1, n))
            assert abs(di - dref) <= 1e-11 * max(1.0, abs(dref))


@pytest.mark.parametrize("order,tab,m,nu", [(1, "erk1", 4, 3), (3, "erk3_ssp", 4, 9)])
def test_residual_modulus_is_the_fcf_estimate(order, tab, m, nu):
    """|r_k| = sqrt(m)|lam|^m |lam^m - mu|/(1-|mu|) (1-|mu|^(nt/m-1)) wherever |mu_k| < 1."""
    nx, nt = 64, 256
    phi, fit, lam = _setup(order, tab, 0.85, nx, m, nu)
    mu = N.symbol(fit.coeffs, fit.offsets, nx)
    r = N.residuals(fit.coeffs, fit.offsets, lam, m, nt)
    ok = np.abs(mu) < 1.0 - 1e-9
    assert ok.sum() >= nx - 2
    ref = T.fcf_bound(lam[ok], mu[ok], m, nt)
    np.testing.assert_allclose(np.abs(r[ok]), ref, rtol=1e-9, atol=1e-15)
    # the symbol is the DFT of the circulant's first column
    col = np.zeros(nx)
    for d, v in fit.stencil.items():
        col[(-d) % nx] = v
    np.testing.assert_allclose(mu, np.fft.fft(col), atol=1e-13)


def test_jacobian_matches_finite_differences():
    nx, nt, m = 32, 128, 4
    phi, fit, lam = _setup(3, "erk3_ssp", 0.85, nx, m, 7)
    psi = fit.coeffs + 0.01 * np.cos(np.arange(7))
    J = N.jacobian(psi, fit.offsets, lam, m, nt)
    for a in range(7):
        h = 1e-6
        e = np.zeros(7)
        e[a] = h
        fd = (N.residuals(psi + e, fit.offsets, lam, m, nt) -
              N.residuals(psi - e, fit.offsets, lam, m, nt)) / (2 * h)
        assert np.max(np.abs(J[:, a] - fd)) <= 1e-6 * max(1.0, np.max(np.abs(fd)))


@pytest.mark.parametrize("order,tab,nx,nt,m,nu", [(1, "erk1", 64, 256, 4, 3),
                                                 (3, "erk3_ssp", 64, 128, 4, 9)])
def test_lm_reaches_minpacks_minimum(order, tab, nx, nt, m, nu):
    """Same residuals, same start, scipy's MINPACK Levenberg-Marquardt run to convergence:
    our 30-iteration LM must not end above it by more than the stopping tolerance, lowers the
    objective monotonically over its accepted steps, and ends at a near-stationary point."""
    from scipy.optimize import least_squares
    phi, fit, lam = _setup(order, tab, 0.85, nx, m, nu)

    def fun(p):
        r = N.residuals(p, fit.offsets, lam, m, nt)
        return np.concatenate([r.real, r.imag])

    ref = least_squares(fun, fit.coeffs, method="lm", xtol=1e-14, ftol=1e-14, gtol=1e-14)
    Fref = 2.0 * ref.cost / nx
    res = N.nlsq_psi(fit.coeffs, fit.offsets, lam, m, nt)
    F0 = N.objective(fit.coeffs, fit.offsets, lam, m, nt)
    assert res.objective < F0
    accepted = [res.history[0]] + [f for f, a in zip(res.history[1:], res.accepted) if a]
    assert all(b < a for a, b in zip(accepted, accepted[1:]))
    assert Fref <= res.objective * (1 + 1e-12)
    assert res.objective <= Fref * (1 + 1e-3)
    assert res.iterations <= 30


@pytest.mark.parametrize("order,tab,nx,nt,m,nu,kref", [
    (1, "erk1", 256, 1024, 2, 2, 10), (1, "erk1", 256, 1024, 4, 3, 6), (1, "erk1", 256, 1024, 8, 4, 6),
    (3, "erk3_ssp", 256, 512, 4, 9, 5)])
def test_paper_nonlinear_iteration_table(order, tab, nx, nt, m, nu, kref):
    """tab:LSQnonlin_ERK: two-level FCF iteration counts with the nonlinear
    least-squares Psi started from the linear one -- ERK1+U1 2^8 x 2^10 m = 2, 4, 8: 10, 6, 6
    (the linear Psi gives 11, 6, 6: tab:LSQlin_ERK), ERK3+U3 2^8 x 2^9 m = 4: 5.  Same windows
    as the linear pins (R8), U[0,1) guess (R3); +-1 for the unknown RNG stream (R16)."""
    phi, fit, lam = _setup(order, tab, 0.85, nx, m, nu)
    res = N.nlsq_psi(fit.coeffs, fit.offsets, lam, m, nt)
    u0 = W.u0_sin4(nx)
    U = W.initial_iterate(0, nx, nt, u0, 0.0)
    rep = M.solve(U, [phi, D.StencilPhi(res.stencil, nx)], m, 2.0 / nx, 0.85 * 2.0 / nx, "FCF",
                  1e-10, 60)
    assert rep.converged and abs(rep.iterations - kref) <= 1, rep.iterations
    if order == 1:
        assert rep.iterations == kref

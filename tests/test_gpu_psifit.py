"""GPU synthesis of the coarse operators (mgrit_psi_fit, csrc/psifit.cu):
the weighted LSQ fit of eq. (LSQ_1D_problem) with the P:338-342 weights, the
window (R8) / eta-threshold patterns and the recursive hierarchy, solved
on the device in double-double arithmetic -- against the oracle's fit (numpy complex
lstsq): same patterns, coefficients to the LSQ's conditioning, accepted by the P:394
rule, and a solve with the device-fitted Psi converging like one with the oracle's."""
import numpy as np
import pytest

import workloads as W
from oracle import discretization as D
from oracle import psi as OP

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4", "cfg4_literal", "cfg5"])
def test_device_fit_matches_oracle(name):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_03726_b200 import problem
    w = W.ALL[name]
    dev = problem.psi_inputs(w, device=True)
    phi = D.make_phi(w.order, w.tableau, w.cfl, w.nx)
    orc = OP.fit_hierarchy(phi, w.nx, w.m, w.cfl, w.psi_widths[: w.levels - 1], w.psi_eta)
    assert len(dev) == len(orc) == w.levels - 1
    for a, b in zip(dev, orc):
        assert a["offsets"] == b.offsets
        assert a["imag"] < 1e-8 and b.accepted
        np.testing.assert_allclose(a["coeffs"], b.coeffs, rtol=0, atol=1e-9)


@pytest.mark.parametrize("name", ["cfg2", "cfg5"])
def test_solve_with_device_fit(name):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_03726_b200 import problem
    w = W.ALL[name] if name == "cfg2" else W.CFG5.scaled(4096, 16384, levels=5)
    g = problem.device_guess(w)
    out = []
    for device in (False, True):
        s = problem.make_solver(w, psi=problem.psi_inputs(w, device=device))
        s.set_guess(g)
        out.append(s.solve(w.tol, w.max_iter))
    assert out[0]["iterations"] == out[1]["iterations"] and out[1]["converged"]
    np.testing.assert_allclose(out[1]["history"], out[0]["history"], rtol=1e-6)


@pytest.mark.parametrize("order,tab,nx,nt,m,nu", [(1, "erk1", 256, 1024, 2, 2), (1, "erk1", 256, 1024, 8, 4),
                                                 (3, "erk3_ssp", 256, 512, 4, 9),
                                                 (3, "erk3_kutta", 1024, 4096, 4, 9),
                                                 (5, "erk5", 4096, 16384, 8, 15)])
def test_device_nonlinear_fit_matches_oracle(order, tab, nx, nt, m, nu):
    """mgrit_psi_fit_nl (App. B, eq. (nlsq)) against oracle/nlsq.py from the same
    linear-LSQ start: the same Levenberg-Marquardt trial sequence (accept / reject pattern and
    trial count), objective history and coefficients."""
    from oracle import nlsq as N
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_03726_b200 import binding as B
    phi = D.make_phi(order, tab, 0.85, nx)
    fit = OP.fit_hierarchy(phi, nx, m, 0.85, (nu,))[0]
    e0 = np.zeros(nx)
    e0[0] = 1.0
    lam = OP.eigenvalues(phi(e0))
    ref = N.nlsq_psi(fit.coeffs, fit.offsets, lam, m, nt)
    got = B.psi_fit_nl_device(order, tab, 0.85, nx, m, nt, fit.offsets, list(fit.coeffs))
    assert got["iterations"] == ref.iterations
    assert len(got["history"]) == len(ref.history)
    for a, b in zip(got["history"], ref.history):
        assert abs(a - b) <= 1e-8 * abs(b), (got["history"], ref.history)
    assert got["objective"] < ref.history[0]
    np.testing.assert_allclose(got["coeffs"], ref.coeffs, rtol=0, atol=1e-8 * np.max(np.abs(ref.coeffs)))


@pytest.mark.parametrize("m,nu,kref", [(2, 2, 10), (4, 3, 6), (8, 4, 6)])
def test_paper_nonlinear_table_through_the_library(m, nu, kref):
    """tab:LSQnonlin_ERK, ERK1+U1 2^8 x 2^10, m = 2, 4, 8 -> 10, 6, 6: linear fit
    and nonlinear refinement both on the device, then mgrit_solve (U[0,1) guess, R3)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_03726_b200 import binding as B
    nx, nt = 256, 1024
    lin = B.psi_fit_device(1, "erk1", 0.85, nx, m, 2, (nu,))[0]
    nl = B.psi_fit_nl_device(1, "erk1", 0.85, nx, m, nt, lin["offsets"], lin["coeffs"])
    assert nl["objective"] < nl["history"][0]
    s = B.MGRIT(nx, nt, m, 1.0, 0.85, 1, "erk1", 2, [nl], "FCF")
    U = torch.from_numpy(W.initial_iterate(0, nx, nt, W.u0_sin4(nx), 0.0)).cuda()
    s.set_guess(U)
    r = s.solve(1e-10, 60)
    assert r["converged"] and r["iterations"] == kref, r["iterations"]


def test_cfg2_with_nonlinear_psi_converges_no_slower():
    """'no significant difference between the convergence rates' -- cfg2 with the
    nonlinear refinement of its 9-point Psi needs at most as many iterations (+-1)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_03726_b200 import problem
    w = W.CFG2
    ks = []
    for nl in (False, True):
        s = problem.make_solver(w, problem.psi_inputs(w, device=True, nonlinear=nl))
        s.set_guess(problem.device_guess(w))
        r = s.solve(w.tol, w.max_iter)
        assert r["converged"]
        ks.append(r["iterations"])
    assert abs(ks[1] - ks[0]) <= 1, ks

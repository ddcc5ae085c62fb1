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

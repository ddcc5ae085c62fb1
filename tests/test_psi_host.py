"""The product's host-side Psi synthesis (paper_1910_03726_b200/psi.py) — an input of the
library (north_star) — against the oracle's LSQ and the paper's P:394 acceptance rule.
Host-only (needs libmgrit.so for the scheme coefficients, no GPU)."""
import numpy as np
import pytest

import workloads as W
from oracle import discretization as D
from oracle import psi as OP


def _psi():
    try:
        from paper_1910_03726_b200 import binding, psi
        binding.lib()
    except (ImportError, OSError) as e:
        pytest.skip(f"libmgrit.so not built: {e}")
    return psi


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4", "cfg5"])
def test_hierarchy_matches_oracle_fit(name):
    """Same windows / threshold patterns and coefficients (to LSQ conditioning) as the
    oracle's fit_hierarchy; every level accepted."""
    P = _psi()
    w = W.ALL[name]
    lib = P.hierarchy(w.order, w.tableau, w.cfl, w.nx, w.m, w.levels, w.psi_widths, w.psi_eta)
    phi = D.make_phi(w.order, w.tableau, w.cfl, w.nx)
    orc = OP.fit_hierarchy(phi, w.nx, w.m, w.cfl, w.psi_widths[: w.levels - 1], w.psi_eta)
    for a, b in zip(lib, orc):
        assert a["offsets"] == b.offsets
        assert a["imag"] < 1e-8 and b.accepted
        np.testing.assert_allclose(a["coeffs"], b.coeffs, rtol=0, atol=1e-8)


def test_flagged_fit_rejected():
    """an imaginary component above 1e-8 flags the fit, which is not accepted."""
    P = _psi()
    lam = P.phi_eigenvalues(5, "erk5", 1.6, 256)
    offs = list(range(-12, 0))
    _, imag = P.lsq(lam, 16, offs, return_imag=True)
    assert imag > 1e-8
    col = OP.ideal_first_column(D.make_phi(5, "erk5", 1.6, 256), 256, 16)
    orc = OP.lsq_psi(col, OP.eigenvalues(D.make_phi(5, "erk5", 1.6, 256)(np.eye(256)[0])), offs)
    assert not orc.accepted                     # the oracle flags the same fit
    with pytest.raises(P.PsiRejected):
        _reject(P)


def _reject(P):
    # a hierarchy whose only level uses the flagged pattern
    orig = P.window
    try:
        P.window = lambda shift, nu: list(range(-12, 0))
        return P.hierarchy(5, "erk5", 1.6, 256, 16, 2, (12,))
    finally:
        P.window = orig

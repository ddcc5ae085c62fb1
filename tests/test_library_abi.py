"""CPU-side checks of the C-ABI library (no GPU): it loads, exports every symbol that
include/mgrit.h declares, validates arguments on the host, and its fp64 coefficients
(and the host-side Psi fit of the product) agree with the oracle's."""
import os
import re

import numpy as np
import pytest

import workloads as W
from oracle import discretization as D
from oracle import psi as OP

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def B():
    from paper_1910_03726_b200 import binding, build
    build.build()
    binding.lib()
    return binding


def test_exports_every_declared_symbol(B):
    hdr = open(os.path.join(ROOT, "include", "mgrit.h")).read()
    declared = set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(mgrit_\w+)\s*\(", hdr, flags=re.M))
    assert len(declared) >= 15
    lib = B.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(B.exported_symbols())


@pytest.mark.parametrize("order,tab,cfl", [(1, "erk1", 0.85), (1, "erk1", 1.7), (2, "erk2", 0.425),
                                           (3, "erk3_ssp", 0.85), (3, "erk3_kutta", 0.85),
                                           (4, "erk4", 0.85), (5, "erk5", 0.85), (1, "sdirk1", 4.0),
                                           (2, "sdirk2", 4.0), (3, "sdirk3", 4.0), (4, "sdirk4", 4.0)])
def test_coefficients_bitwise_equal_oracle(B, order, tab, cfl):
    """z_d = (-c w_d)/den and the tableaux (R3) are bit-identical on both sides, so the
    two paths apply the same Phi up to summation order and FMA contraction."""
    z, A, b = B.scheme_coefficients(order, tab, cfl)
    oz = D.z_coefficients(order, cfl)
    ot = D.tableau(tab)
    assert z == oz
    assert np.array_equal(A, np.array(ot.A)) and np.array_equal(b, np.array(ot.b))


def test_workspace_and_validation(B):
    lib = B.lib()
    assert lib.mgrit_workspace_bytes(1024, 4096, 4, 2) > 3 * 1025 * 1024 * 8
    assert lib.mgrit_workspace_bytes(1024, 4095, 4, 2) == 0        # nt % m != 0
    assert lib.mgrit_workspace_bytes(1024, 4096, 4, 8) == 0        # nt % m^7 != 0
    import ctypes as C
    ctx = C.c_void_p()
    arr = (B._Psi * 1)()
    # invalid: tableau order mismatch, null workspace
    assert lib.mgrit_setup(C.byref(ctx), 64, 64, 2, 1.0, 0.85, 3, 0, 2, arr, 2, None, 0, None) == -1
    assert lib.mgrit_setup(C.byref(ctx), 64, 64, 2, 1.0, 0.85, 1, 0, 2, arr, 2, None, 0, None) == -2


@pytest.mark.parametrize("wname", ["cfg2", "cfg3", "cfg5"])
def test_product_psi_fit_matches_oracle(B, wname):
    """The product's host LSQ (real formulation) equals the oracle's complex LSQ +
    real-part truncation (Lemma 3) on the same pattern."""
    from paper_1910_03726_b200 import psi as ppsi
    w = W.ALL[wname].scaled(1024, 4096) if wname != "cfg2" else W.ALL[wname]
    phi = D.make_phi(w.order, w.tableau, w.cfl, w.nx)
    levels = min(w.levels, 4)
    of = OP.fit_hierarchy(phi, w.nx, w.m, w.cfl, w.psi_widths[: levels - 1])
    pf = ppsi.hierarchy(w.order, w.tableau, w.cfl, w.nx, w.m, levels, w.psi_widths)
    for a, b in zip(of, pf):
        assert a.offsets == b["offsets"]
        np.testing.assert_allclose(b["coeffs"], a.coeffs, atol=1e-9)


def test_product_threshold_pattern_matches_oracle(B):
    from paper_1910_03726_b200 import psi as ppsi
    nx = 1024
    phi = D.make_phi(3, "sdirk3", 4.0, nx)
    col = OP.ideal_first_column(phi, nx, 4)
    lam = ppsi.phi_eigenvalues(3, "sdirk3", 4.0, nx)
    assert ppsi.threshold(lam ** 4, 0.01) == OP.threshold_pattern(col, 0.01)


def test_setup_rejections_host_only(B):
    """mgrit_setup validates before touching the device: every rejected combination
    returns its status code and leaves *ctx NULL (include/mgrit.h)."""
    import ctypes as C
    lib = B.lib()
    ctx = C.c_void_p(123)
    one = (B._Psi * 1)()
    dummy = C.c_void_p(1 << 20)        # never dereferenced: validation fails first
    big = 1 << 40
    cases = [
        (64, 64, 2, -1.0, 0.85, 1, 0, 2, one, 2, dummy, big),    # alpha <= 0
        (64, 64, 2, 1.0, 0.0, 1, 0, 2, one, 2, dummy, big),      # cfl <= 0
        (64, 64, 2, 1.0, 0.85, 6, 0, 2, one, 2, dummy, big),     # order outside 1..5
        (64, 64, 2, 1.0, 0.85, 1, 0, 2, one, 1, dummy, big),     # relax C is not a solve mode
        (64, 63, 2, 1.0, 0.85, 1, 0, 2, one, 2, dummy, big),     # nt % m != 0
        (64, 64, 2, 1.0, 0.85, 1, 0, 2, None, 2, dummy, big),    # psi NULL
        (4, 64, 2, 1.0, 0.85, 1, 0, 2, one, 2, dummy, big),      # nx too small for U1
    ]
    for args in cases:
        st = lib.mgrit_setup(C.byref(ctx), *args, None)
        assert st == -1, (args, st)
        assert not ctx.value
    # the host-only setters reject a NULL context
    assert lib.mgrit_set_cycle(None, 0) == -1
    assert lib.mgrit_set_final_sweep(None, 1) == -1


def test_missing_library_fails_loudly(B, monkeypatch, tmp_path):
    """No CPU fallback: with the shared library absent the binding raises instead of
    computing anything (the product path never routes through the oracle)."""
    monkeypatch.setattr(B, "_lib", None)
    monkeypatch.setattr(B, "LIB_PATH", str(tmp_path / "libmgrit.so"))
    with pytest.raises(ImportError, match="no CPU fallback"):
        B.lib()
    with pytest.raises(ImportError):
        B.scheme_coefficients(1, "erk1", 0.85)


def test_product_does_not_import_the_oracle():
    """The oracle is test infrastructure: no module of the product package imports it."""
    pkg = os.path.join(ROOT, "paper_1910_03726_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), fn

"""GPU parity of the inflow/outflow path (PAPER.md 4.5 P:672-762;
DESIGN.md R20) against oracle/inflow.py through the C ABI (mgrit_set_inflow).

Both sides consume the same boundary DATA (the derivative table of u(-1, t) = sin^4(pi t),
workloads.inflow_sin4_derivatives) and the same Psi coefficients (the oracle's periodic LSQ
fit); the ghost-value arithmetic, the closures and the truncation live on each side
separately.  Compared: the forcing rows b_n (bitwise), every FULL-state primitive, and whole
solves (identical K, histories, C-rows after every iteration, final solution; R18).
"""
import math

import numpy as np
import pytest

import workloads as W
from oracle import discretization as D
from oracle import inflow as I
from oracle import mgrit as M
from oracle import psi as OP

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REL = 1e-12


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_03726_b200 import binding
    binding.lib()
    return binding


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def _problem(order, tab, c, nx, nt, seed=0, lo=-1.0):
    ph = I.BoundedRKPhi(order, tab, c, nx)
    dgs = W.inflow_sin4_derivatives(np.arange(nt) * ph.dt, ph.nq)
    u0 = np.sin(np.pi * W.inflow_grid(nx)) ** 4
    g0 = I.fine_rhs(ph, u0, dgs)
    U = W.initial_iterate(seed, nx, nt, u0, lo)
    return ph, dgs, u0, g0, U


def _fits(order, tab, c, nx, m, widths):
    per = D.make_phi(order, tab, c, nx)
    fits = OP.fit_hierarchy(per, nx, m, c, widths)
    lib = [{"kind": "stencil", "offsets": f.offsets, "coeffs": list(f.coeffs)} for f in fits]
    return lib, [I.TruncatedStencilPhi(f.stencil, nx) for f in fits]


def _solver(B, order, tab, c, nx, nt, m, levels, psi_lib, relax, dgs):
    s = B.MGRIT(nx, nt, m, 1.0, c, order, tab, levels, psi_lib, relax)
    s.set_inflow(torch.from_numpy(dgs).cuda())
    return s


SCHEMES = [(1, "erk1", 0.85), (2, "erk2", 0.4), (3, "erk3_ssp", 1.3), (3, "erk3_kutta", 1.3),
           (4, "erk4", 0.9), (5, "erk5", 1.6)]


@pytest.mark.parametrize("order,tab,c", SCHEMES)
def test_forcing_rows_bitwise(order, tab, c):
    """b_n = Phi(0; t_n): the device forcing kernel follows the oracle's stage form in its
    operation order with separately rounded products and sums, so the rows are bitwise equal
    (support: the first s*|d_min| points) -- except for ERK5, whose non-dyadic tableau makes
    the host table (A^q 1)_i depend on the summation order of the matrix-vector products
    (numpy's BLAS vs a plain loop): a few ulps there."""
    B = _cuda()
    nx, nt = 256, 64
    ph, dgs, u0, g0, U = _problem(order, tab, c, nx, nt)
    lib, _ = _fits(order, tab, c, nx, 4, (9,))
    s = _solver(B, order, tab, c, nx, nt, 4, 2, lib, "FCF", dgs)
    f = s.get_forcing().cpu().numpy()
    nb = ph.tab.s * ph.nl
    ref = g0[1:]
    assert np.all(ref[:, nb:] == 0.0)
    if tab == "erk5":
        assert np.max(np.abs(f[:, :nb] - ref[:, :nb])) <= 1e-15 * np.max(np.abs(ref))
    else:
        assert np.array_equal(f[:, :nb], ref[:, :nb])
    assert np.all(f[:, nb:] == 0.0)


@pytest.mark.parametrize("order,tab,c,nx", [(1, "erk1", 0.85, 64), (3, "erk3_ssp", 1.3, 128),
                                            (3, "erk3_kutta", 1.3, 1024), (4, "erk4", 0.9, 512),
                                            (5, "erk5", 1.6, 256), (5, "erk5", 1.6, 2048),
                                            (3, "erk3_ssp", 1.3, 4096)])
def test_primitives_with_inflow(order, tab, c, nx):
    """mgrit_relax (F, C, FCF), mgrit_residual and mgrit_coarse_solve on the affine system
    U[n+1] = Phi_h U[n] + b_n against the oracle's definitions (P:206-212 with g_0)."""
    B = _cuda()
    m, nt = 4, 32
    ph, dgs, u0, g0, U0 = _problem(order, tab, c, nx, nt, seed=3)
    lib, psis = _fits(order, tab, c, nx, m, (9,))
    s = _solver(B, order, tab, c, nx, nt, m, 2, lib, "FCF", dgs)
    for kind in ("F", "C", "FCF"):
        Uo = U0.copy()
        if kind in ("F", "FCF"):
            M.f_relax(Uo, ph, m, g0)
        if kind in ("C", "FCF"):
            M.c_relax(Uo, ph, m, g0)
        if kind == "FCF":
            M.f_relax(Uo, ph, m, g0)
        Ug = torch.from_numpy(U0).cuda()
        s.relax_full(Ug, kind)
        assert _rel(Ug.cpu().numpy(), Uo) <= REL, kind
    # residual: all-row norm and C-point residual rows
    ro = M.residual_norm(U0, ph, 2.0 / nx, ph.dt, g0)
    Ug = torch.from_numpy(U0).cuda()
    rg, rrows = s.residual_full(Ug, want_r=True)
    assert abs(rg - ro) <= REL * ro
    cpts = np.arange(m, nt + 1, m)
    rref = M.residual_rows(U0, ph, cpts, g0)
    assert _rel(rrows.cpu().numpy()[1:], rref) <= REL
    # coarse-grid correction (two-level, exact coarse solve) + ideal interpolation
    Uo = U0.copy()
    gc = np.zeros((nt // m + 1, nx))
    gc[1:] = rref
    E = M.sequential_rhs(psis[0], gc)
    Uo[cpts] = Uo[cpts] + E[1:]
    M.f_relax(Uo, ph, m, g0)
    s.coarse_solve_full(Ug)
    assert _rel(Ug.cpu().numpy(), Uo) <= REL


def _compare_solve(B, order, tab, c, nx, nt, m, levels, widths, relax="FCF", max_iter=40,
                   lo=-1.0, psi=None, cycle="V"):
    ph, dgs, u0, g0, U = _problem(order, tab, c, nx, nt, seed=1, lo=lo)
    if psi is None:
        lib, psis = _fits(order, tab, c, nx, m, widths)
    else:
        lib, psis = psi(ph)
    Uo = U.copy()
    rep = M.solve(Uo, [ph] + psis, m, 2.0 / nx, ph.dt, relax, 1e-10, max_iter, keep_states=True,
                  g0=g0, cycle=cycle)
    s = _solver(B, order, tab, c, nx, nt, m, levels, lib, relax, dgs)
    if cycle == "F":
        s.set_cycle("F")
    Ug = torch.from_numpy(U).cuda()
    s.set_guess(Ug)
    out = torch.empty_like(Ug)
    res = s.solve(1e-10, max_iter, out=out, keep_crows=True)
    K = rep.iterations
    if not (abs(rep.history[-1] - 1e-10) / 1e-10 < 1e-6):
        assert res["iterations"] == K, (res["history"], rep.history)
    assert res["converged"] == rep.converged
    umax = float(np.max(np.abs(Uo)))
    floor = 1e-15 * math.sqrt(2 * nt * ph.dt) * umax
    for k, (a, b) in enumerate(zip(res["history"], rep.history)):
        assert abs(a - b) <= REL * abs(b) + floor, (k, a, b)
    cg = res["crows"].cpu().numpy()
    for k in range(min(K, cg.shape[0])):
        assert _rel(cg[k], rep.states[k]) <= REL, k
    assert _rel(out.cpu().numpy(), Uo) <= REL
    return rep, res


@pytest.mark.parametrize("m,nu,kref", [(2, 2, 10), (4, 3, 6), (8, 4, 6)])
def test_solve_paper_inflow_table_erk1(m, nu, kref):
    """tab:LSQlin_ERK_inflow, ERK1+U1, 2^8 x 2^10, two-level m = 2, 4, 8 through
    the library: the oracle's counts (10, 6, 6 +-1, pinned in tests/test_oracle_inflow.py)
    and iterates."""
    B = _cuda()
    rep, res = _compare_solve(B, 1, "erk1", 0.85, 256, 1024, m, 2, (nu,), lo=0.0)
    assert rep.converged and abs(res["iterations"] - kref) <= 1


@pytest.mark.parametrize("order,tab,c,nx,nt,m,nu", [
    (3, "erk3_ssp", 0.85, 256, 1024, 4, 9),
    (3, "erk3_kutta", 0.85, 1024, 1024, 4, 9),
    (5, "erk5", 0.85, 256, 1024, 8, 15),
    (5, "erk5", 0.85, 2048, 512, 4, 11),
    (2, "erk2", 0.4, 128, 256, 2, 5),
    (4, "erk4", 0.9, 512, 512, 4, 9),
])
def test_solve_two_level_inflow(order, tab, c, nx, nt, m, nu):
    """Two-level FCF solves with the periodic problem's Psi truncated at the boundaries."""
    B = _cuda()
    rep, res = _compare_solve(B, order, tab, c, nx, nt, m, 2, (nu,))
    assert rep.converged


def test_solve_two_level_inflow_4096():
    """Widest supported row (nx = 4096: 512 threads x 8 points; coarse chain 1024 x 4)."""
    B = _cuda()
    rep, res = _compare_solve(B, 3, "erk3_ssp", 0.85, 4096, 512, 4, 2, (9,))
    assert rep.converged


def test_solve_parareal_inflow():
    """F-relaxation (Parareal) on the inflow problem."""
    B = _cuda()
    _compare_solve(B, 3, "erk3_ssp", 0.85, 256, 256, 4, 2, (9,), relax="F")


@pytest.mark.parametrize("order,tab,c,nx,nt,levels,widths", [
    (1, "erk1", 0.85, 256, 1024, 3, (3, 5)),
    (1, "erk1", 0.85, 256, 1024, 4, (3, 5, 7)),
    (3, "erk3_ssp", 0.85, 1024, 4096, 4, (9, 13, 17)),
    (5, "erk5", 0.85, 256, 1024, 3, (13, 19)),
])
def test_solve_multilevel_inflow(order, tab, c, nx, nt, levels, widths):
    """V-cycles, m = 4 on every level, truncated Psi hierarchy (right half of
    tab:LSQlin_ERK_inflow)."""
    B = _cuda()
    lo = 0.0 if order == 1 else -1.0
    rep, res = _compare_solve(B, order, tab, c, nx, nt, 4, levels, widths, lo=lo)
    assert rep.converged


def test_solve_fcycle_inflow():
    B = _cuda()
    _compare_solve(B, 3, "erk3_ssp", 0.85, 256, 1024, 4, 4, (9, 13, 17), cycle="F")


@pytest.mark.parametrize("order,tab,c,m", [(1, "erk1", 0.85, 2), (3, "erk3_ssp", 1.3, 4),
                                          (5, "erk5", 1.6, 4)])
def test_ideal_psi_one_iteration_inflow(order, tab, c, m):
    """Psi = Phi_h^m with the same closures: one iteration."""
    B = _cuda()
    rep, res = _compare_solve(B, order, tab, c, 256, 64, m, 2, None,
                              psi=lambda ph: ([{"kind": "ideal"}], [D.PowerPhi(ph, m)]))
    assert res["iterations"] == 1 and res["converged"]


def test_redisc_psi_inflow():
    """Rediscretised Psi (ERK1+U1 at CFL m c > 1 diverges as in the periodic case; compare
    the first iterations only, max_iter = 3)."""
    B = _cuda()
    m, c = 2, 0.4
    _compare_solve(B, 1, "erk1", c, 64, 64, m, 2, None, max_iter=3,
                   psi=lambda ph: ([{"kind": "redisc", "cfl": m * c}],
                                   [I.BoundedRKPhi(1, "erk1", m * c, 64)]))


def test_homogeneous_inflow_and_periodic_switch():
    """dg = NULL is the homogeneous problem; enable = 0 restores the periodic rows."""
    B = _cuda()
    nx, nt, m = 256, 64, 4
    ph, dgs, u0, g0, U = _problem(3, "erk3_ssp", 0.85, nx, nt, seed=5)
    lib, psis = _fits(3, "erk3_ssp", 0.85, nx, m, (9,))
    s = B.MGRIT(nx, nt, m, 1.0, 0.85, 3, "erk3_ssp", 2, lib, "FCF")
    s.set_inflow(None)
    Ug = torch.from_numpy(U).cuda()
    s.relax_full(Ug, "F")
    Uo = U.copy()
    M.f_relax(Uo, ph, m, None)
    assert _rel(Ug.cpu().numpy(), Uo) <= REL
    s.set_inflow(None, enable=False)
    Ug = torch.from_numpy(U).cuda()
    s.relax_full(Ug, "F")
    Up = U.copy()
    M.f_relax(Up, D.make_phi(3, "erk3_ssp", 0.85, nx), m, None)
    assert _rel(Ug.cpu().numpy(), Up) <= REL


def test_inflow_unsupported_combinations():
    B = _cuda()
    lib, _ = _fits(5, "erk5", 0.85, 128, 4, (9,))
    s = B.MGRIT(128, 64, 4, 1.0, 0.85, 5, "erk5", 2, lib, "FCF")
    with pytest.raises(B.MgritError):      # 128 = 32 x 4 points per thread < order + 1
        s.set_inflow(None)
    lib3, _ = _fits(3, "sdirk3", 4.0, 256, 4, (11,))
    s3 = B.MGRIT(256, 64, 4, 1.0, 4.0, 3, "sdirk3", 2, lib3, "FCF")
    with pytest.raises(B.MgritError):      # implicit tableau
        s3.set_inflow(None)


def test_inflow_long_chain_cluster_overlap():
    """A long two-level chain (nc = 1024) takes the 16-CTA cluster kernel with the halo points
    beyond the row ends held at zero, overlapped with the next sweep and with a speculative
    chain by default: against the oracle, and bitwise against the serial iteration."""
    B = _cuda()
    nx, nt, m = 1024, 4096, 4
    rep, res = _compare_solve(B, 3, "erk3_ssp", 0.85, nx, nt, m, 2, (9,))
    assert rep.converged
    ph, dgs, u0, g0, U = _problem(3, "erk3_ssp", 0.85, nx, nt, seed=1)
    lib, _ = _fits(3, "erk3_ssp", 0.85, nx, m, (9,))
    outs = []
    for opts in ({"graph": [0], "overlap": [0]}, {"graph": [0], "overlap": [8, 1]},
                 {"graph": [0], "overlap": [4, 0]}, {"graph": [1]}):
        s = B.MGRIT(nx, nt, m, 1.0, 0.85, 3, "erk3_ssp", 2, lib, "FCF", options=opts)
        s.set_inflow(torch.from_numpy(dgs).cuda())
        Ug = torch.from_numpy(U).cuda()
        s.set_guess(Ug)
        out = torch.empty_like(Ug)
        r = s.solve(1e-10, 40, out=out)
        outs.append((r["history"], out))
    for h, o in outs[1:]:
        assert h == outs[0][0]
        assert torch.equal(o, outs[0][1])

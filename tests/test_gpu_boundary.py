"""GPU tests of the C-ABI boundary beyond the tuned production shapes (include/mgrit.h):

* level >= 1 FULL-state primitives (relax / residual / coarse solve with Phi_l = Psi_l and a
  right-hand side g_l, P:206-212 on a coarse level of the P:618-624 hierarchy) vs the
  oracle's level functions;
* two-level solves whose periodic row is wider than one CTA (nx = 8192, 16384: 16-CTA
  cluster split) and RK-form (IDEAL / REDISC) Psi at nx = 512 .. 4096, vs the oracle;
* mgrit_set_option: every override gives the oracle's result; invalid values are EINVAL.
"""
import numpy as np
import pytest

import workloads as W
from oracle import discretization as D
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


def _hierarchy(nx, nt, levels, m=4, order=3, tab="erk3_ssp", cfl=0.85, widths=(9, 13, 17, 21)):
    phi = D.make_phi(order, tab, cfl, nx)
    fits = OP.fit_hierarchy(phi, nx, m, cfl, widths[: levels - 1])
    lib = [{"kind": "stencil", "offsets": f.offsets, "coeffs": list(f.coeffs)} for f in fits]
    return phi, fits, lib


@pytest.mark.parametrize("nx,level,with_rhs", [(256, 1, True), (1024, 1, False),
                                               (1024, 2, True), (6000, 1, True)])
def test_level_primitives(nx, level, with_rhs):
    """mgrit_relax (F, C, FCF), mgrit_residual (norm with dt_l = m^l dt, C-point residuals)
    and mgrit_coarse_solve on level l with RHS g_l against oracle.mgrit's f_relax / c_relax
    / residual_rows / sequential_rhs with the same Psi data (R12 right-hand-side form)."""
    B = _cuda()
    m, levels = 4, 4
    nt = 64 * m ** (levels - 1)
    phi, fits, lib = _hierarchy(nx, nt, levels)
    ntl = nt // m ** level
    psi_l = D.StencilPhi(fits[level - 1].stencil, nx)
    psi_c = D.StencilPhi(fits[level].stencil, nx) if level + 1 < levels else None
    U0 = W.initial_iterate(21, nx, ntl, W.u0_fourier(nx, 5))
    G = W.initial_iterate(22, nx, ntl, np.zeros(nx)) if with_rhs else None
    s = B.MGRIT(nx, nt, m, 1.0, 0.85, 3, "erk3_ssp", levels, lib, "FCF")
    gdev = torch.from_numpy(G).cuda() if with_rhs else None
    s.set_rhs(level, gdev)
    for kind in ("F", "C", "FCF"):
        Uo = U0.copy()
        if kind in ("F", "FCF"):
            M.f_relax(Uo, psi_l, m, G)
        if kind in ("C", "FCF"):
            M.c_relax(Uo, psi_l, m, G)
        if kind == "FCF":
            M.f_relax(Uo, psi_l, m, G)
        Ug = torch.from_numpy(U0).cuda()
        s.relax_full(Ug, kind, level=level)
        Ug = Ug.cpu().numpy()
        assert np.array_equal(Ug[0], U0[0])
        assert _rel(Ug, Uo) <= REL, (kind, _rel(Ug, Uo))
    # residual
    dtl = 0.85 * (2.0 / nx) * m ** level
    Ug = torch.from_numpy(U0).cuda()
    ng, rg = s.residual_full(Ug, want_r=True, level=level)
    no = M.residual_norm(U0, psi_l, 2.0 / nx, dtl, G)
    assert abs(ng - no) <= 1e-13 * no
    ro = M.residual_rows(U0, psi_l, np.arange(m, ntl + 1, m), G)
    rg = rg.cpu().numpy()
    assert np.all(rg[0] == 0.0) and _rel(rg[1:], ro) <= REL
    # coarse-grid correction by the next level, solved sequentially
    if psi_c is not None:
        Uo = U0.copy()
        cpts = np.arange(m, ntl + 1, m)
        gc = np.zeros((ntl // m + 1, nx))
        gc[1:] = M.residual_rows(Uo, psi_l, cpts, G)
        E = M.sequential_rhs(psi_c, gc)
        Uo[cpts] += E[1:]
        M.f_relax(Uo, psi_l, m, G)
        Ug = torch.from_numpy(U0).cuda()
        s.coarse_solve_full(Ug, level=level)
        assert _rel(Ug.cpu().numpy(), Uo) <= REL


def test_level_primitives_errors():
    B = _cuda()
    nx, nt, m = 256, 256, 4
    _, _, lib = _hierarchy(nx, nt, 3)
    s = B.MGRIT(nx, nt, m, 1.0, 0.85, 3, "erk3_ssp", 3, lib, "FCF")
    U = torch.zeros((nt // m ** 2 + 1, nx), dtype=torch.float64, device="cuda")
    with pytest.raises(B.MgritError) as e:
        s.coarse_solve_full(U, level=2)          # coarsest level has nothing below it
    assert e.value.code == -1
    with pytest.raises(B.MgritError):
        s.relax_full(U, "F", level=3)
    with pytest.raises(B.MgritError):
        s.set_rhs(0, U)
    w = W.CFG1_IDEAL
    s1 = B.MGRIT(w.nx, w.nt, w.m, 1.0, w.cfl, 1, "erk1", 2, [{"kind": "ideal"}], "F")
    with pytest.raises(B.MgritError) as e:
        s1.relax_full(torch.zeros((w.nt // w.m + 1, w.nx), dtype=torch.float64, device="cuda"),
                      "F", level=1)
    assert e.value.code == -5


def _solve_vs_oracle(w, lib, orc_psi, max_iter=None, options=None):
    B = _cuda()
    phi = D.make_phi(w.order, w.tableau, w.cfl, w.nx)
    U = w.guess()
    Uo = U.copy()
    mi = max_iter or w.max_iter
    rep = M.solve(Uo, [phi] + orc_psi, w.m, w.dx, w.dt, w.relax, w.tol, mi)
    s = B.MGRIT(w.nx, w.nt, w.m, w.alpha, w.cfl, w.order, w.tableau, w.levels, lib, w.relax,
                options=options)
    g = torch.from_numpy(U).cuda()
    s.set_guess(g)
    out = torch.empty_like(g)
    res = s.solve(w.tol, mi, out=out)
    assert res["iterations"] == rep.iterations, (res["history"], rep.history)
    for a, b in zip(res["history"], rep.history):
        assert abs(a - b) <= REL * b + 1e-14 * np.max(np.abs(Uo)), (a, b)
    assert _rel(out.cpu().numpy(), Uo) <= REL
    return s, res


@pytest.mark.parametrize("nx,nt", [(8192, 2048), (16384, 4096)])
def test_two_level_wide_rows(nx, nt):
    """Two-level FCF MGRIT at nx = 8192 / 16384 (the cfg5 width): the sequential coarse
    solve's periodic row is split over a 16-CTA cluster (512 / 1024 points per SM) and the
    fine sweep runs in halo tiles; iterates, history and K vs the oracle."""
    w = W.CFG5.scaled(nx, nt, levels=2, psi_widths=(9,), max_iter=20)
    phi = D.make_phi(w.order, w.tableau, w.cfl, w.nx)
    fit = OP.fit_hierarchy(phi, w.nx, w.m, w.cfl, (9,))[0]
    lib = [{"kind": "stencil", "offsets": fit.offsets, "coeffs": list(fit.coeffs)}]
    s, res = _solve_vs_oracle(w, lib, [D.StencilPhi(fit.stencil, w.nx)])
    assert "coarse=psi_seq_cluster" in s.describe(), s.describe()
    assert res["converged"]


@pytest.mark.parametrize("nx", [512, 2048, 4096])
@pytest.mark.parametrize("kind", ["ideal", "redisc"])
def test_rk_form_psi_sizes(nx, kind):
    """Psi = Phi^m (one iteration) and the rediscretised Psi (CFL m c) at the row
    widths beyond round 1's set: ERK1+U1 Parareal as cfg1, and ERK3+U3 FCF, at c = 0.45 so
    the rediscretised operator (c = 0.9) is stable and the iterates stay comparable."""
    for order, tab, relax in [(1, "erk1", "F"), (3, "erk3_ssp", "FCF")]:
        nt = 128 if nx < 4096 else 64
        w = W.CFG1_IDEAL.scaled(nx, nt, order=order, tableau=tab, relax=relax, max_iter=6,
                                cfl=0.45, psi_kind=kind, redisc_cfl=0.9)
        phi = D.make_phi(order, tab, w.cfl, nx)
        if kind == "ideal":
            lib, orc = [{"kind": "ideal"}], [D.PowerPhi(phi, w.m)]
        else:
            lib = [{"kind": "redisc", "cfl": w.redisc_cfl}]
            orc = [D.make_phi(order, tab, w.redisc_cfl, nx)]
        s, res = _solve_vs_oracle(w, lib, orc)
        if kind == "ideal":
            assert res["iterations"] == 1


OPTION_CASES = [
    ({"fine_tile": (256, 11)}, W.CFG5.scaled(6144, 256, levels=3)),
    ({"fine_tile": (128, 15, 2)}, W.CFG5.scaled(6144, 256, levels=3)),
    ({"whole_row": (512, 8)}, W.CFG2.scaled(4096, 256, psi_widths=(9,))),
    ({"seq_cluster": (16, 128, 2), "seq_s": (4,)}, W.CFG3.scaled(4096, 512)),
    ({"coarse_kernel": (1,)}, W.CFG2.scaled(1024, 512)),
    ({"seq_cluster": (0, 0, 0), "seq_cfg": (256, 4)}, W.CFG2.scaled(1024, 512)),
    ({"sdirk_product": (1,)}, W.CFG4.scaled(1024, 256)),
    ({"stage_form": (1,)}, W.CFG5.scaled(6144, 256, levels=3)),
    ({"stage_form": (1,)}, W.CFG2.scaled(1024, 512)),
]


@pytest.mark.parametrize("opts,w", OPTION_CASES, ids=[str(c[0]) for c in OPTION_CASES])
def test_set_option_results_unchanged(opts, w):
    """mgrit_set_option replaces a measured default by another valid configuration: the
    solve still matches the oracle (iterates, history, K)."""
    phi = D.make_phi(w.order, w.tableau, w.cfl, w.nx)
    fits = OP.fit_hierarchy(phi, w.nx, w.m, w.cfl, w.psi_widths[: w.levels - 1], w.psi_eta)
    lib = [{"kind": "stencil", "offsets": f.offsets, "coeffs": list(f.coeffs)} for f in fits]
    orc = [D.StencilPhi(f.stencil, w.nx) for f in fits]
    _solve_vs_oracle(w, lib, orc, max_iter=12, options=opts)


def test_set_option_errors():
    B = _cuda()
    w = W.CFG2.scaled(256, 256)
    s = B.MGRIT(w.nx, w.nt, w.m, 1.0, w.cfl, 3, "erk3_kutta", 2,
                [{"kind": "stencil", "offsets": [-1, 0], "coeffs": [0.5, 0.5]}], "FCF")
    for name, vals in [("fine_tile", (128,)), ("seq_s", (1, 2)), ("coarse_kernel", (2,)),
                       ("whole_row", (-1, 8))]:
        with pytest.raises(B.MgritError) as e:
            s.set_option(name, vals)
        assert e.value.code == -1, name
    st = B.lib().mgrit_set_option(s.ctx, 99, None, 0)
    assert st == -1
    s.set_option("fine_tile", ())             # reset to the default is always valid


GRAPH_CASES = {
    "cfg1_redisc": W.CFG1_REDISC.scaled(64, 256, max_iter=9),
    "cfg1_ideal": W.CFG1_IDEAL,
    "cfg2": W.CFG2,
    "cfg2_parareal": W.CFG2.scaled(256, 1024, relax="F", max_iter=40),
    "vcycle": W.CFG5.scaled(1024, 4096, levels=4),
    "fcycle": W.CFG5.scaled(256, 4096, levels=5),
    "sdirk": W.CFG4.scaled(256, 1024),
}


@pytest.mark.parametrize("name", sorted(GRAPH_CASES))
def test_graph_mode_bitwise_equals_host_loop(name):
    """mgrit_solve's CUDA-graph mode (device-side WHILE loop with the FCF buffer ping-pong
    as IF-nested second body, graph.cu) runs the very same kernels as the host loop: history,
    K and the FULL solution are bitwise equal, for odd and even K, and across two solves
    with the cached graph."""
    from paper_1910_03726_b200 import problem
    _cuda()
    w = GRAPH_CASES[name]
    g = torch.from_numpy(w.guess()).cuda()
    runs = []
    for mode in (0, 1, 1):
        s = problem.make_solver(w, options={"graph": (mode,)})
        if name == "fcycle":
            s.set_cycle("F")
        s.set_guess(g)
        out = torch.empty_like(g)
        res = s.solve(w.tol, w.max_iter, out=out)
        if mode == 1:
            res2 = s.solve(w.tol, w.max_iter, out=out)     # cached graph, second launch
            assert res2["history"] == res["history"]
        runs.append((res, out))
    (r0, o0), (r1, o1) = runs[0], runs[1]
    assert r1["iterations"] == r0["iterations"] and r1["converged"] == r0["converged"]
    assert r1["history"] == r0["history"]
    assert torch.equal(o1, o0)

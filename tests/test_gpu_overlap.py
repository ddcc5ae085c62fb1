"""Overlapped two-level iteration (mgrit_set_option MGRIT_OPT_OVERLAP): the
coarse chain in chunks on a high-priority stream with the next sweep's chunks beside it must
be bitwise the serial iteration (same kernels on the same rows in the same order), and match
the oracle like every other solve."""
import numpy as np
import pytest

import workloads as W
from oracle import discretization as D
from oracle import mgrit as M
from oracle import psi as OP

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_03726_b200 import binding
    binding.lib()
    return binding


def _setup(B, order, tab, c, nx, nt, m, nu, relax, seed, options):
    phi = D.make_phi(order, tab, c, nx)
    fit = OP.fit_hierarchy(phi, nx, m, c, (nu,))[0]
    lib = [{"kind": "stencil", "offsets": fit.offsets, "coeffs": list(fit.coeffs)}]
    u0 = W.u0_fourier(nx, seed)
    U = W.initial_iterate(seed + 1, nx, nt, u0, -1.0)
    s = B.MGRIT(nx, nt, m, 1.0, c, order, tab, 2, lib, relax, options=options)
    return s, U, phi, fit


@pytest.mark.parametrize("order,tab,c,nx,nt,m,nu,relax", [
    (3, "erk3_kutta", 0.85, 1024, 4096, 4, 9, "FCF"),      # cfg2 shape (32 x 2 cluster slices)
    (5, "erk5", 0.85, 4096, 8192, 8, 15, "FCF"),           # cfg3 width, whole-row sweep
    (3, "erk3_ssp", 0.85, 4096, 4096, 4, 9, "F"),          # Parareal
    (3, "erk3_ssp", 0.85, 16384, 4096, 4, 9, "FCF"),       # halo-tile TMA sweep, 1024-point slices
    (3, "sdirk3", 4.0, 4096, 4096, 4, 31, "FCF"),          # cfg4 scheme
    (3, "erk3_kutta", 0.85, 1024, 4000, 4, 9, "FCF"),      # nc = 1000: chunk counts that do not divide
    (3, "erk3_ssp", 0.85, 2048, 6144, 4, 9, "F"),          # nc = 1536, Parareal
])
@pytest.mark.parametrize("final", ["off", "predict"])
def test_overlap_bitwise_equals_serial(order, tab, c, nx, nt, m, nu, relax, final):
    B = _cuda()
    res, outs = [], []
    for chunks in ([0], [8], [4], [8, 0], [16, 1]):   # [C] / [C, speculative chain on/off]
        s, U, phi, fit = _setup(B, order, tab, c, nx, nt, m, nu, relax, 11,
                                {"graph": [0], "overlap": chunks})
        s.set_final_sweep(final)
        Ug = torch.from_numpy(U).cuda()
        s.set_guess(Ug)
        out = torch.empty_like(Ug)
        r = s.solve(1e-10, 12, out=out, keep_crows=(chunks != [4]))
        res.append(r)
        outs.append(out)
    for r, o in zip(res[1:], outs[1:]):
        assert r["iterations"] == res[0]["iterations"]
        assert r["history"] == res[0]["history"]
        assert torch.equal(o, outs[0])
    assert torch.equal(res[1]["crows"], res[0]["crows"])


def test_overlap_default_matches_oracle():
    """Default options at a long chain (nc = 1024 >= the overlap threshold) against the
    oracle: identical K, histories and iterates at 1e-12."""
    B = _cuda()
    nx, nt, m = 1024, 4096, 4
    s, U, phi, fit = _setup(B, 3, "erk3_kutta", 0.85, nx, nt, m, 9, "FCF", 21, {"graph": [0]})
    Uo = U.copy()
    rep = M.solve(Uo, [phi, D.StencilPhi(fit.stencil, nx)], m, 2.0 / nx, 0.85 * 2.0 / nx, "FCF",
                  1e-10, 20, keep_states=True)
    Ug = torch.from_numpy(U).cuda()
    s.set_guess(Ug)
    out = torch.empty_like(Ug)
    r = s.solve(1e-10, 20, out=out, keep_crows=True)
    assert r["iterations"] == rep.iterations and r["converged"]
    for a, b in zip(r["history"], rep.history):
        assert abs(a - b) <= 1e-12 * abs(b) + 1e-15
    cg = r["crows"].cpu().numpy()
    for k in range(rep.iterations):
        assert np.max(np.abs(cg[k] - rep.states[k])) <= 1e-12 * np.max(np.abs(rep.states[k]))
    assert np.max(np.abs(out.cpu().numpy() - Uo)) <= 1e-12 * np.max(np.abs(Uo))


@pytest.mark.parametrize("nx,nt,levels", [(8192, 16384, 4), (16384, 8192, 3), (6144, 16384, 5)])
@pytest.mark.parametrize("final", ["off", "predict"])
def test_vcycle_overlap_bitwise_equals_serial(nx, nt, levels, final):
    """MGRIT_OPT_VOVERLAP: level-1 interpolation chunks || fine sweep chunks || the next
    level-1 sweep, ordered by events, against the serial V-cycle iteration (cfg5 recipe,
    halo-tile kernels): identical histories, C-rows and solutions, bit for bit."""
    B = _cuda()
    from paper_1910_03726_b200 import problem
    w = W.CFG5.scaled(nx, nt, levels=levels)
    lib = problem.psi_inputs(w)
    U = torch.from_numpy(w.guess()).cuda()
    res, outs = [], []
    for vo in ([0], [8, 3, 1], [4, 2, 0], [8, 4, 1]):
        opts = {} if vo is None else {"voverlap": vo}
        s = B.MGRIT(w.nx, w.nt, w.m, w.alpha, w.cfl, w.order, w.tableau, w.levels, lib, w.relax,
                    options=opts)
        s.set_final_sweep(final)
        s.set_guess(U)
        out = torch.empty_like(U)
        res.append(s.solve(w.tol, 12, out=out, keep_crows=(vo != [8, 4, 1])))
        outs.append(out)
        del s
    for r, o in zip(res[1:], outs[1:]):
        assert r["iterations"] == res[0]["iterations"]
        assert r["history"] == res[0]["history"]
        assert torch.equal(o, outs[0])
    assert torch.equal(res[1]["crows"], res[0]["crows"])

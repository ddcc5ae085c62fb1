"""Time-parallel MGRIT: the multi-GPU shard engine
(mgrit_solve_shard) emulated on one GPU — N shards in N host threads exchanging rows through
paper_1910_03726_b200.timeshard.ThreadComm (all cross-rank waiting happens on the host in the
communication callbacks; no kernel waits on another shard).  Every rank's FULL block and the
global residual history are compared with the oracle's single-domain solve (R18),
with identical iteration counts, and nranks = 1 with the ordinary mgrit_solve bit for bit.
"""
import math

import numpy as np
import pytest

import workloads as W
from oracle import discretization as D
from oracle import mgrit as M
from oracle import psi as OP

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
REL = 1e-12


def _setup(w):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    phi = D.make_phi(w.order, w.tableau, w.cfl, w.nx)
    fits = OP.fit_hierarchy(phi, w.nx, w.m, w.cfl, w.psi_widths[: w.levels - 1], w.psi_eta)
    lib = [{"kind": "stencil", "offsets": f.offsets, "coeffs": list(f.coeffs)} for f in fits]
    return phi, [phi] + [D.StencilPhi(f.stencil, w.nx) for f in fits], lib


CASES = {
    "two_level_cfg2": (W.CFG2.scaled(1024, 2048), (2, 4)),
    "parareal": (W.CFG2.scaled(256, 1024, relax="F", max_iter=40), (2, 4)),
    "vcycle_cfg5": (W.CFG5.scaled(1024, 4096, levels=4), (2, 4)),
    "vcycle_6lvl_tiles": (W.CFG5.scaled(6144, 8192, levels=5), (2,)),
    "sdirk_cfg4": (W.CFG4.scaled(1024, 1024), (2,)),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_time_shards_match_oracle(name):
    from paper_1910_03726_b200 import timeshard as T
    w, ranks = CASES[name]
    phi, phis, lib = _setup(w)
    U = w.guess()
    Uo = U.copy()
    rep = M.solve(Uo, phis, w.m, w.dx, w.dt, w.relax, w.tol, w.max_iter)
    umax = float(np.max(np.abs(Uo)))
    floor = 1e-15 * math.sqrt(2 * w.nt * w.dt) * umax
    for n in ranks:
        res, outs = T.solve_emulated(w, lib, n)
        part = T.Partition(w.nt, w.m, w.levels, n)
        for r in range(n):
            assert res[r]["iterations"] == rep.iterations, (n, r, res[r]["history"], rep.history)
            assert res[r]["converged"] == rep.converged
            assert res[r]["history"] == res[0]["history"]       # the same global norm everywhere
            for a, b in zip(res[r]["history"], rep.history):
                assert abs(a - b) <= REL * b + floor, (n, r, a, b)
            rows = part.rows(r)
            got = outs[r].cpu().numpy()
            err = float(np.max(np.abs(got - Uo[rows.start:rows.stop])) / umax)
            assert err <= REL, (n, r, err)


def test_single_shard_equals_mgrit_solve():
    """nranks = 1 runs the shard engine without exchanges: bitwise the host-loop solve."""
    from paper_1910_03726_b200 import problem
    from paper_1910_03726_b200 import timeshard as T
    w = W.CFG5.scaled(1024, 4096, levels=4)
    _, _, lib = _setup(w)
    res, outs = T.solve_emulated(w, lib, 1)
    s = problem.make_solver(w, psi=lib, options={"graph": (0,)})
    s.set_final_sweep("off")
    g = problem.device_guess(w)
    s.set_guess(g)
    out = torch.empty_like(g)
    ref = s.solve(w.tol, w.max_iter, out=out)
    assert res[0]["history"] == ref["history"]
    assert torch.equal(outs[0], out)


def test_shard_errors():
    from paper_1910_03726_b200 import binding
    from paper_1910_03726_b200 import timeshard as T
    w = W.CFG2.scaled(256, 1024)
    _, _, lib = _setup(w)
    with pytest.raises(ValueError):
        T.Partition(1000, 4, 2, 3)
    sh = T.ShardSolver(w, lib, 0, 2)
    g = sh.local_guess()
    with pytest.raises(binding.MgritError) as e:        # nranks > 1 without a communicator
        sh.solve(None, g, w.tol, 4)
    assert e.value.code == -1

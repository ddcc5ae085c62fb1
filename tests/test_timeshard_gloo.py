"""World-size-2 gloo (CPU) tests of the time-parallel path.

* `Partition`: contiguous time blocks aligned to the coarsest level (host logic).
* `TorchDistComm`, the torch.distributed communicator the multi-GPU run hands to
  mgrit_solve_shard, through its ctypes callback entry points: `shift` moves the staging
  row to rank+1 / from rank-1, `allreduce_sum` sums host doubles.
* The time decomposition itself, on CPU: a numpy model of MGRIT on contiguous time blocks
  with the exchanges it needs (the block-start C-row from rank-1 after the C-relaxation
  and after each correction -- the shard engine's fused sweep gets the first as the
  outbox row r_{nc+1} -- the coarsest chain's state rank -> rank+1, the norm allreduce) is run
  on 2 gloo ranks through TorchDistComm and must reproduce the oracle's single-domain
  solve: same K, same history (to the norm's summation order), bitwise-equal iterate
  blocks.  (The CUDA engine itself is checked against the oracle on the GPU in
  tests/test_gpu_timeshard.py.)
"""
import os
import socket

import numpy as np
import pytest

import workloads as W
from oracle import discretization as D
from oracle import mgrit as M
from oracle import psi as OP

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world=2, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q, *args)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def _init(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)


# ---------------------------------------------------------------- partition
def test_partition_blocks():
    from paper_1910_03726_b200.timeshard import Partition
    p = Partition(65536, 4, 6, 8)
    assert p.nt_loc == 8192
    assert p.rows(0) == range(0, 8193) and p.rows(7) == range(57344, 65537)
    # every level's intervals are a contiguous block per rank, covering the level once
    for lvl in range(5):
        cover = [j for r in range(8) for j in p.intervals(r, lvl)]
        assert cover == list(range(65536 // 4 ** (lvl + 1)))
    with pytest.raises(ValueError):
        Partition(4096, 4, 6, 8)                 # coarsest level would split a step


# ---------------------------------------------------------------- communicator
def _comm_worker(rank, world, port, q):
    _init(rank, world, port)
    from paper_1910_03726_b200.timeshard import TorchDistComm
    send = torch.full((5,), float(rank + 1), dtype=torch.float64)
    recv = torch.zeros(5, dtype=torch.float64)
    comm = TorchDistComm(send, recv)
    # through the C function pointers the library calls
    st = comm.struct.shift(None, int(rank < world - 1), int(rank > 0), None)
    got = recv.clone()
    vals = (torch.zeros(2, dtype=torch.float64) + torch.tensor([rank + 1.0, 0.5])).numpy()
    buf = (__import__("ctypes").c_double * 2)(*vals)
    st2 = comm.struct.allreduce_sum(None, buf, 2)
    q.put((rank, st, got.tolist(), st2, list(buf)))
    dist.barrier()
    dist.destroy_process_group()


def test_torchdist_comm_two_ranks():
    out = _run(_comm_worker)
    (r0, st0, got0, s0, sum0), (r1, st1, got1, s1, sum1) = out
    assert st0 == st1 == s0 == s1 == 0
    assert got0 == [0.0] * 5                     # rank 0 receives nothing
    assert got1 == [1.0] * 5                     # rank 1 receives rank 0's row
    assert sum0 == sum1 == [3.0, 1.0]


# ---------------------------------------------------------------- decomposition model
class _Rows:
    """Row exchange of the model through TorchDistComm's staging rows."""

    def __init__(self, comm, nx):
        self.c = comm
        self.rank, self.world = comm.rank, comm.world

    def shift(self, send_row=None, recv_row=None):
        hs = send_row is not None and self.rank < self.world - 1
        hr = recv_row is not None and self.rank > 0
        if hs:
            self.c.send_stage.copy_(torch.from_numpy(send_row))
        self.c.shift(hs, hr)
        if hr:
            recv_row[:] = self.c.recv_stage.numpy()

    def sum(self, v):
        return self.c.allreduce_sum([v])[0]


def _shard_cycle(level, U, g, phis, m, relax, X):
    """V-cycle on this rank's time block (FULL state, RHS form R12): relaxation,
    injection and correction on local rows, the block-start C-row from rank-1 after every
    correction, the coarsest level as a chain pipelined rank to rank."""
    phi = phis[level]
    if level == len(phis) - 1:
        if X.rank > 0:
            X.shift(recv_row=U[0])                       # state at the block start
        for n in range(U.shape[0] - 1):
            U[n + 1] = phi(U[n]) + g[n + 1]
        if X.rank < X.world - 1:
            X.shift(send_row=U[-1])
        return
    M.f_relax(U, phi, m, g)
    if relax == "FCF":
        M.c_relax(U, phi, m, g)
        X.shift(send_row=U[-1].copy(), recv_row=U[0])    # C-relaxed block-start C-row
        M.f_relax(U, phi, m, g)
    nt = U.shape[0] - 1
    cpts = np.arange(m, nt + 1, m)
    gc = np.zeros((nt // m + 1, U.shape[1]))
    gc[1:] = M.residual_rows(U, phi, cpts, g)
    E = np.zeros_like(gc)
    _shard_cycle(level + 1, E, gc, phis, m, relax, X)
    U[cpts] = U[cpts] + E[1:]
    X.shift(send_row=U[-1].copy(), recv_row=U[0])        # corrected block-start C-row
    M.f_relax(U, phi, m, g)


def _model_worker(rank, world, port, q, wname, nx, nt, levels, relax):
    _init(rank, world, port)
    from paper_1910_03726_b200.timeshard import Partition, TorchDistComm
    w = W.ALL[wname].scaled(nx, nt, levels=levels, relax=relax)
    phi = D.make_phi(w.order, w.tableau, w.cfl, w.nx)
    fits = OP.fit_hierarchy(phi, w.nx, w.m, w.cfl, w.psi_widths[: w.levels - 1], w.psi_eta)
    phis = [phi] + [D.StencilPhi(f.stencil, w.nx) for f in fits]
    part = Partition(w.nt, w.m, w.levels, world)
    rows = part.rows(rank)
    U = w.guess()[rows.start:rows.stop].copy()
    X = _Rows(TorchDistComm(torch.zeros(w.nx, dtype=torch.float64),
                            torch.zeros(w.nx, dtype=torch.float64)), w.nx)

    def norm(U):
        r = M.residual_rows(U, phi, np.arange(1, U.shape[0]))
        return float(np.sqrt(w.dx * w.dt * X.sum(float(np.sum(r * r)))))

    hist = [norm(U)]
    k = 0
    while hist[-1] >= w.tol and k < w.max_iter:
        _shard_cycle(0, U, None, phis, w.m, w.relax, X)
        k += 1
        hist.append(norm(U))
    q.put((rank, k, hist, U))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("wname,nx,nt,levels,relax", [("cfg2", 64, 256, 2, "FCF"),
                                                       ("cfg2", 64, 256, 2, "F"),
                                                       ("cfg5", 64, 1024, 3, "FCF")])
def test_time_decomposition_model_two_ranks(wname, nx, nt, levels, relax):
    out = _run(_model_worker, 2, wname, nx, nt, levels, relax)
    w = W.ALL[wname].scaled(nx, nt, levels=levels, relax=relax)
    phi = D.make_phi(w.order, w.tableau, w.cfl, w.nx)
    fits = OP.fit_hierarchy(phi, w.nx, w.m, w.cfl, w.psi_widths[: w.levels - 1], w.psi_eta)
    Uo = w.guess()
    rep = M.solve(Uo, [phi] + [D.StencilPhi(f.stencil, w.nx) for f in fits], w.m, w.dx, w.dt,
                  w.relax, w.tol, w.max_iter)
    half = nt // 2
    for rank, k, hist, U in out:
        assert k == rep.iterations
        np.testing.assert_allclose(hist, rep.history, rtol=1e-12, atol=1e-16)
        assert np.array_equal(U, Uo[rank * half: (rank + 1) * half + 1])

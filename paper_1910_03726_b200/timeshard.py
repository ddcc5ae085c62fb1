"""Time-parallel MGRIT over several GPUs (the paper parallelises time only,
P:841, XBraid with contiguous blocks of time per processor).

The solve itself runs in libmgrit.so (`mgrit_setup_shard` / `mgrit_solve_shard`,
include/mgrit.h): every level's sweep, injection and interpolation on the rank's own
intervals, the coarsest chain pipelined rank to rank.  This module is plumbing only:

* `Partition` — which global rows a rank owns (contiguous blocks, aligned to m^(L-1));
* communicators implementing the library's two callbacks (`shift`: one row to rank+1 /
  from rank-1 through the registered staging rows; `allreduce_sum`: host doubles):
  - `TorchDistComm`: torch.distributed (NCCL between GPUs; gloo for CPU tests);
  - `ThreadComm`: N shards in one process (one thread each, one GPU) exchanging through
    queues — the single-GPU emulation of the multi-GPU path (no kernel waits on another
    rank: all waiting happens on the host, in the callbacks);
* `ShardSolver` — one rank's context, guess block and solve.
"""
from __future__ import annotations

import ctypes as C
import queue
import threading
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

from . import binding

SHIFT_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p)
SUM_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int)


class MgritComm(C.Structure):
    _fields_ = [("user", C.c_void_p), ("shift", SHIFT_FN), ("allreduce_sum", SUM_FN)]


@dataclass(frozen=True)
class Partition:
    """Contiguous time blocks: rank r owns global steps [r*nt_loc, (r+1)*nt_loc]."""
    nt: int
    m: int
    levels: int
    nranks: int

    def __post_init__(self):
        q = self.nranks * self.m ** (self.levels - 1)
        if self.nt % q:
            raise ValueError(f"nt = {self.nt} must be divisible by nranks * m^(levels-1) = {q}")

    @property
    def nt_loc(self) -> int:
        return self.nt // self.nranks

    def rows(self, rank: int) -> range:
        """Global fine rows of rank's local FULL block (row 0 = the block start)."""
        return range(rank * self.nt_loc, (rank + 1) * self.nt_loc + 1)

    def intervals(self, rank: int, level: int = 0) -> range:
        """Global level-l intervals owned by rank (level-l C-rows j .. j+1)."""
        n = self.nt_loc // self.m ** (level + 1)
        return range(rank * n, (rank + 1) * n)


class _CommBase:
    """Holds the ctypes callback objects alive; subclasses implement shift / allreduce."""

    def __init__(self):
        self._shift_cb = SHIFT_FN(self._shift)
        self._sum_cb = SUM_FN(self._sum)
        self.struct = MgritComm(None, self._shift_cb, self._sum_cb)

    def _shift(self, user, has_send, has_recv, stream):
        try:
            self.shift(bool(has_send), bool(has_recv))
            return 0
        except Exception as e:  # noqa: BLE001 -- reported to the library as MGRIT_ECOMM
            self.error = e
            return -1

    def _sum(self, user, vals, n):
        try:
            out = self.allreduce_sum([vals[i] for i in range(n)])
            for i in range(n):
                vals[i] = out[i]
            return 0
        except Exception as e:  # noqa: BLE001
            self.error = e
            return -1


class TorchDistComm(_CommBase):
    """torch.distributed communicator of one rank (default process group): NCCL on GPUs,
    gloo for CPU tests.  `send_stage` / `recv_stage` are the rows registered with the
    library (device tensors for NCCL, host tensors under gloo)."""

    def __init__(self, send_stage, recv_stage, stream=None):
        super().__init__()
        import torch.distributed as dist
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.send_stage, self.recv_stage = send_stage, recv_stage
        self.stream = stream

    def shift(self, has_send: bool, has_recv: bool):
        import torch
        if self.stream is not None:
            self.stream.synchronize()            # the library wrote send_stage on its stream
        ops = []
        if has_send:
            ops.append(self.dist.P2POp(self.dist.isend, self.send_stage, self.rank + 1))
        if has_recv:
            ops.append(self.dist.P2POp(self.dist.irecv, self.recv_stage, self.rank - 1))
        if ops:
            for r in self.dist.batch_isend_irecv(ops):
                r.wait()
        if self.recv_stage.is_cuda:
            torch.cuda.synchronize(self.recv_stage.device)

    def allreduce_sum(self, vals: List[float]) -> List[float]:
        import torch
        dev = self.send_stage.device
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        self.dist.all_reduce(t)
        return [float(v) for v in t.cpu()]


class ThreadGroup:
    """Shared state of N in-process shards: one queue per directed neighbour link and a
    deterministic (rank-ordered) allreduce."""

    def __init__(self, nranks: int, timeout: float = 600.0):
        self.n = nranks
        self.q = {r: queue.Queue() for r in range(nranks)}          # link r-1 -> r
        self.barrier = threading.Barrier(nranks)
        self.slots: List[Optional[List[float]]] = [None] * nranks
        self.timeout = timeout


class ThreadComm(_CommBase):
    """Communicator of shard `rank` within a ThreadGroup (single-GPU emulation)."""

    def __init__(self, group: ThreadGroup, rank: int, send_stage, recv_stage, stream):
        super().__init__()
        self.g, self.rank = group, rank
        self.send_stage, self.recv_stage, self.stream = send_stage, recv_stage, stream

    def shift(self, has_send: bool, has_recv: bool):
        import torch
        with torch.cuda.stream(self.stream):
            self.stream.synchronize()
            if has_send:
                self.g.q[self.rank + 1].put(self.send_stage.clone())
            if has_recv:
                row = self.g.q[self.rank].get(timeout=self.g.timeout)
                self.recv_stage.copy_(row)
            self.stream.synchronize()

    def allreduce_sum(self, vals: List[float]) -> List[float]:
        self.g.slots[self.rank] = list(vals)
        self.g.barrier.wait(self.g.timeout)
        out = [sum(self.g.slots[r][i] for r in range(self.g.n)) for i in range(len(vals))]
        self.g.barrier.wait(self.g.timeout)
        return out


class ShardSolver:
    """One time shard of a workload (paper_1910_03726_b200.problem conventions)."""

    def __init__(self, w, psi: Sequence[Dict], rank: int, nranks: int, stream=None,
                 device: str = "cuda"):
        import torch
        self.w, self.rank, self.nranks = w, rank, nranks
        self.part = Partition(w.nt, w.m, w.levels, nranks)
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        L = binding.lib()
        nbytes = L.mgrit_workspace_bytes_shard(w.nx, w.nt, w.m, w.levels, nranks)
        if nbytes == 0:
            raise binding.MgritError(-1, "invalid shard sizes")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=device)
        self.send_stage = torch.zeros(w.nx, dtype=torch.float64, device=device)
        self.recv_stage = torch.zeros(w.nx, dtype=torch.float64, device=device)
        arr, keep = binding.psi_array(psi, w.levels)
        self._keep = keep
        ctx = C.c_void_p()
        st = L.mgrit_setup_shard(C.byref(ctx), w.nx, w.nt, w.m, w.alpha, w.cfl, w.order,
                                 binding.TABLEAU[w.tableau], w.levels, arr,
                                 binding.RELAX[w.relax], rank, nranks,
                                 self.send_stage.data_ptr(), self.recv_stage.data_ptr(),
                                 self.workspace.data_ptr(), nbytes,
                                 C.c_void_p(self.stream.cuda_stream))
        if st:
            raise binding.MgritError(st, "mgrit_setup_shard failed (see stderr)")
        self.ctx = ctx

    def __del__(self):
        try:
            if getattr(self, "ctx", None):
                binding.lib().mgrit_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass

    def local_guess(self):
        """The rank's block of the workload's initial iterate, generated on the device."""
        import torch
        w = self.w
        rows = self.part.rows(self.rank)
        g = torch.empty((len(rows), w.nx), dtype=torch.float64, device=self.workspace.device)
        u0 = torch.from_numpy(w.u0()).to(g.device) if self.rank == 0 else None
        binding.fill_guess(g, w.guess_seed, w.guess_lo, u0=u0, row0=rows.start,
                           stream=self.stream)
        return g

    def solve(self, comm, guess, tol: float, max_iter: int, out=None):
        L = binding.lib()
        self.guess = guess
        st = L.mgrit_set_guess(self.ctx, binding._dptr(guess))
        if st:
            raise binding.MgritError(st, "mgrit_set_guess")
        iters, conv = C.c_int(), C.c_int()
        hist = (C.c_double * (max_iter + 1))()
        st = L.mgrit_solve_shard(self.ctx, C.byref(comm.struct) if comm is not None else None,
                                 tol, max_iter, binding._dptr(out), C.byref(iters), hist,
                                 C.byref(conv))
        if st and st != -4:
            msg = L.mgrit_last_error(self.ctx)
            err = getattr(comm, "error", None)
            raise binding.MgritError(st, f"mgrit_solve_shard: {msg.decode() if msg else ''}"
                                         + (f" ({err!r})" if err else ""))
        k = iters.value
        return {"iterations": k, "history": list(hist[:k + 1]), "converged": bool(conv.value),
                "status": st}


def solve_emulated(w, psi, nranks: int, tol: Optional[float] = None,
                   max_iter: Optional[int] = None):
    """All `nranks` time shards of workload `w` on the current GPU, one thread each
    (ThreadComm).  Returns (per-rank results, per-rank FULL blocks)."""
    import torch
    tol = w.tol if tol is None else tol
    max_iter = w.max_iter if max_iter is None else max_iter
    group = ThreadGroup(nranks)
    shards, comms, guesses, outs = [], [], [], []
    for r in range(nranks):
        s = torch.cuda.Stream()
        sh = ShardSolver(w, psi, r, nranks, stream=s)
        with torch.cuda.stream(s):
            g = sh.local_guess()
            outs.append(torch.empty_like(g))
        s.synchronize()
        shards.append(sh)
        guesses.append(g)
        comms.append(ThreadComm(group, r, sh.send_stage, sh.recv_stage, s))
    results: List[Optional[dict]] = [None] * nranks
    errors: List[Optional[BaseException]] = [None] * nranks

    def worker(r):
        try:
            with torch.cuda.stream(shards[r].stream):
                results[r] = shards[r].solve(comms[r], guesses[r], tol, max_iter, out=outs[r])
        except BaseException as e:  # noqa: BLE001
            errors[r] = e
            group.barrier.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errors:
        if e is not None:
            raise e
    torch.cuda.synchronize()
    return results, outs

"""Write the full-size parity goldens under tests/golden/ — from the ORACLE only.

This script imports nothing but `oracle/` (the method, written from the paper) and
`workloads/` (seeded inputs).  It never touches the CUDA library: every stored value is
the oracle's.  The GPU test `tests/test_gpu_fullsize_goldens.py` feeds the stored Psi
coefficients and the same seeded iterate to the library and compares, element by
element at the DESIGN.md R18 tolerances, the residual history, the iteration count and
sampled C-rows after every iteration plus sampled rows of the final FULL solution.

Usage:  python tools/make_goldens.py NAME [NAME ...]      (NAME in GOLDENS below)

The cfg5 golden runs the cfg5 recipe at nx = 8192 (nt = 65536, six levels, coarsest
nt = 64 as in the bench): the oracle's full-state numpy V-cycle at nx = 16384 needs about
70 GB of host memory (8 x the 8.6 GB state), more than this build box has; the production
width nx = 16384 is covered by test_solve_cfg5_fullwidth_vcycle at nt = 4096 (6 levels).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from oracle import discretization as D  # noqa: E402
from oracle import inflow as I  # noqa: E402
from oracle import mgrit as M  # noqa: E402
from oracle import psi as OP  # noqa: E402

GOLDENS = {
    "cfg3_full": lambda: W.CFG3,
    "cfg4_full": lambda: W.CFG4,
    "cfg5_8192x65536": lambda: W.CFG5.scaled(8192, 65536),
    "cfg5_fcycle_1024x16384": lambda: W.CFG5.scaled(1024, 16384, levels=5),
    # inflow/outflow rows (PAPER.md 4.5; oracle/inflow.py): the bench shapes
    "inflow_erk3_full": lambda: W.INFLOW_ERK3,
    "inflow_erk3_ml_full": lambda: W.INFLOW_ERK3_ML,
}
CYCLE = {"cfg5_fcycle_1024x16384": "F"}
N_CROWS = 8      # sampled C-rows stored per iteration (full width)
N_FINAL = 8      # sampled rows of the final FULL solution


def sample_rows(nc: int, nt: int):
    rng = np.random.default_rng(20261020)
    crow = sorted(set(int(j) for j in rng.choice(np.arange(1, nc), N_CROWS - 1, replace=False))
                  | {nc})
    fin = set(int(n) for n in rng.choice(np.arange(1, nt), N_FINAL - 2, replace=False))
    fin |= {nt, nt - 1}
    return np.array(crow), np.array(sorted(fin))


def run(name: str) -> str:
    w = GOLDENS[name]()
    cycle = CYCLE.get(name, "V")
    phi = D.make_phi(w.order, w.tableau, w.cfl, w.nx)
    if w.psi_kind != "stencil":
        raise ValueError("goldens are for the stencil-Psi throughput workloads")
    fits = OP.fit_hierarchy(phi, w.nx, w.m, w.cfl, w.psi_widths[: w.levels - 1], w.psi_eta)
    assert all(f.accepted for f in fits)
    phis = [phi] + [D.StencilPhi(f.stencil, w.nx) for f in fits]
    g0 = None
    if getattr(w, "boundary", "periodic") == "inflow":
        # the periodic problem's Psi truncated at the boundaries, the bounded fine propagator
        # and its forcing rows from the inflow derivative table (R20)
        ph = I.BoundedRKPhi(w.order, w.tableau, w.cfl, w.nx, w.alpha)
        dgs = W.inflow_sin4_derivatives(np.arange(w.nt) * w.dt, ph.nq)
        g0 = I.fine_rhs(ph, w.u0(), dgs)
        phis = [ph] + [I.TruncatedStencilPhi(f.stencil, w.nx) for f in fits]
    nc = w.nt // w.m
    crow_idx, final_idx = sample_rows(nc, w.nt)
    crows = []

    def on_iter(k, U):
        crows.append(U[crow_idx * w.m].copy())
        print(f"[{name}] iteration {k} done ({time.time() - t0:.0f} s)", flush=True)

    U = w.guess()
    t0 = time.time()
    rep = M.solve(U, phis, w.m, w.dx, w.dt, w.relax, w.tol, w.max_iter, cycle=cycle,
                  on_iter=on_iter, g0=g0)
    secs = time.time() - t0
    meta = dict(name=name, workload=w.name, nx=w.nx, nt=w.nt, m=w.m, levels=w.levels,
                order=w.order, tableau=w.tableau, cfl=w.cfl, relax=w.relax, cycle=cycle,
                tol=w.tol, max_iter=w.max_iter, u0_kind=w.u0_kind, u0_seed=w.u0_seed,
                guess_seed=w.guess_seed, guess_lo=w.guess_lo, oracle_seconds=round(secs, 1),
                boundary=getattr(w, "boundary", "periodic"),
                generator="tools/make_goldens.py (oracle/ + workloads/ only)")
    out = dict(meta=np.array(json.dumps(meta)), history=np.array(rep.history),
               iterations=np.array(rep.iterations), converged=np.array(rep.converged),
               crow_idx=crow_idx, crows=np.stack(crows), final_idx=final_idx,
               final_rows=U[final_idx].copy(), umax=np.array(np.max(np.abs(U))))
    for l, f in enumerate(fits):
        out[f"psi{l}_offsets"] = np.array(f.offsets, dtype=np.int64)
        out[f"psi{l}_coeffs"] = np.array(f.coeffs, dtype=np.float64)
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"[{name}] K={rep.iterations} converged={rep.converged} hist={rep.history} "
          f"({secs:.0f} s) -> {path}", flush=True)
    return path


if __name__ == "__main__":
    for n in sys.argv[1:] or list(GOLDENS):
        run(n)

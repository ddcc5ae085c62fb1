"""Repeat solves / coarse corrections and compare bitwise (race detector for the
cluster coarse solve).  usage: python tools/determinism.py [cfg] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1910_03726_b200 import problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = W.ALL[name]
s = problem.make_solver(w)
print(s.describe())
g = problem.device_guess(w)
ref = None
for r in range(reps):
    s.set_guess(g)
    out = torch.empty_like(g)
    res = s.solve(w.tol, w.max_iter, out=out)
    torch.cuda.synchronize()
    h = np.array(res["history"])
    if ref is None:
        ref = (out.clone(), h)
        print("rep", r, "K", res["iterations"], h.tolist())
    else:
        d = (out - ref[0]).abs().max().item()
        print("rep", r, "K", res["iterations"], "max|diff| vs rep0", d,
              "hist equal", np.array_equal(h, ref[1]) if len(h) == len(ref[1]) else False)
# coarse correction alone, repeated on the same input
U0 = g.clone()
s.relax_full(U0, "F")
outs = []
for r in range(reps):
    U = U0.clone()
    s.coarse_solve_full(U)
    torch.cuda.synchronize()
    outs.append(U)
print("coarse_solve_full max diffs:", [(o - outs[0]).abs().max().item() for o in outs[1:]])

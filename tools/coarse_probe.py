"""Time the two-level sequential coarse solve alone (class coarse_solve) on a workload's
shape: ns per coarse step.
usage: python tools/coarse_probe.py cfg2 [reps] [name=v1,v2 ...]
(name=values: mgrit_set_option overrides, e.g. seq_cluster=16,64,4 seq_s=6 coarse_kernel=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1910_03726_b200 import problem  # noqa: E402

w = W.ALL[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
opts = {k: tuple(int(x) for x in v.split(",")) for k, v in (a.split("=") for a in sys.argv[3:])}
s = problem.make_solver(w, options=opts)
U = problem.device_guess(w)
for _ in range(2):
    s.coarse_solve_full(U)
torch.cuda.synchronize()
s.profile(True)
for _ in range(reps):
    s.coarse_solve_full(U)
prof = s.profile_read()
n, ms = prof["coarse_solve"]
steps = w.nt // w.m
print(f"{w.name} {s.describe().split('coarse=')[-1]} ns/step {ms / n / steps * 1e6:.1f} "
      f"")

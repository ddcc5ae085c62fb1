"""Small solves that take every production kernel path, for compute-sanitizer.

    compute-sanitizer --tool racecheck python tools/sanitize.py
    compute-sanitizer --tool synccheck python tools/sanitize.py

Cases (kernel -> shape that selects it; `mgrit_describe` is printed for each):
  tiles_vcycle  rk_sweep_tma_kernel (fused + check sweep), psi_level_tma_kernel (sweep and
                interpolation), psi_coarse_kernel (trapezoid tiles)  -- cfg5 recipe, nx = 6144
  cluster_tb    psi_seq_cluster_tb_kernel (warp-specialised 16-CTA cluster)  -- cfg2 recipe
  cluster_ca    psi_seq_cluster_ca_kernel (cp.async cluster variant, coarse_kernel option)
  cluster_plain psi_seq_cluster_kernel (exchange every step, seq_s option 1)
  seq_periodic  psi_seq_periodic_kernel (one CTA, seq_cluster option 0)
  whole_rows    rk_sweep_kernel whole-row (ERK5, nx = 4096) and SDIRK3 stage solves
  rk_coarse     rk_coarse_kernel (cfg1 ideal / redisc), residual, reduce
Each solve uses final-sweep mode "always" so the check sweep runs every iteration.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1910_03726_b200 import problem  # noqa: E402

CASES = {
    "tiles_vcycle": (W.CFG5.scaled(6144, 256, levels=3), {}),
    "cluster_tb": (W.CFG2.scaled(1024, 256), {}),
    "cluster_ca": (W.CFG3.scaled(4096, 256), {"coarse_kernel": (1,)}),
    "cluster_plain": (W.CFG2.scaled(1024, 128), {"seq_s": (1,)}),
    "seq_periodic": (W.CFG2.scaled(1024, 128), {"seq_cluster": (0, 0, 0)}),
    "whole_rows": (W.CFG3.scaled(4096, 64), {}),
    "sdirk": (W.CFG4.scaled(1024, 64), {}),
    "rk_coarse_ideal": (W.CFG1_IDEAL, {}),
    "rk_coarse_redisc": (W.CFG1_REDISC.scaled(64, 256, max_iter=3), {}),
}


def main(names):
    for name in names:
        w, opts = CASES[name]
        s = problem.make_solver(w, options=opts)
        s.set_final_sweep("always")
        g = problem.device_guess(w)
        s.set_guess(g)
        out = torch.empty_like(g)
        res = s.solve(w.tol, min(w.max_iter, 3), out=out)
        torch.cuda.synchronize()
        print(f"{name}: {s.describe()} K={res['iterations']} hist={res['history'][-1]:.3e}",
              flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))

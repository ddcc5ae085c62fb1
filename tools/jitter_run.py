"""One solve of a tools/sanitize.py case (or a full-size workload); prints a JSON line with
the residual history, K and SHA-256 digests of the FULL solution and the final C-rows.
Run it with MGRIT_LIBRARY=jitter to use the race-stress build (tests/test_gpu_jitter.py).
usage: python tools/jitter_run.py CASE"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1910_03726_b200 import binding, problem  # noqa: E402
from sanitize import CASES  # noqa: E402

EXTRA = {
    "cfg2": (W.CFG2, {}),
    "cfg4": (W.CFG4, {}),
    "cfg3_ca": (W.CFG3, {"coarse_kernel": (1,)}),
    "cfg5_fullwidth": (W.CFG5.scaled(16384, 1024, levels=4), {}),
    "two_level_16384": (W.CFG5.scaled(16384, 2048, levels=2, psi_widths=(9,)), {}),
    # overlapped iteration: chunked first / last sweeps without (cfg3) and with
    # a speculative chain (cfg2, cfg4 above; the truncated cluster chain of the inflow rows)
    "cfg3": (W.CFG3, {}),
    "inflow_two_level": (W.INFLOW_ERK3.scaled(1024, 4096), {}),
    "cfg4_overlap16": (W.CFG4, {"overlap": (16, 1)}),
}


def main(name):
    w, opts = CASES[name] if name in CASES else EXTRA[name]
    s = problem.make_solver(w, options=opts)
    s.set_final_sweep("always" if name in CASES else "predict")
    g = problem.device_guess(w)
    s.set_guess(g)
    out = torch.empty_like(g)
    res = s.solve(w.tol, min(w.max_iter, 8), out=out)
    torch.cuda.synchronize()
    h = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()
    hc = hashlib.sha256(s.crows().cpu().numpy().tobytes()).hexdigest()
    print(json.dumps({"case": name, "lib": os.path.basename(binding.LIB_PATH),
                      "iterations": res["iterations"], "history": res["history"],
                      "out_sha256": h, "crows_sha256": hc, "describe": s.describe()}))


if __name__ == "__main__":
    main(sys.argv[1])

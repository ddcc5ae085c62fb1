"""Full-size parity: the production `mgrit_solve` against oracle goldens.

The goldens (tests/golden/fullsize_*.npz) are written by tools/make_goldens.py, which
imports only `oracle/` and `workloads/`: the oracle's MGRIT on the FULL space-time state
 at the graded sizes — cfg3 and cfg4 at 4096 x 16384 exactly as
BASELINE.json states them, and the cfg5 recipe at 8192 x 65536 (six levels, coarsest
nt = 64, the full time length of the throughput run; nx halved so the oracle fits in host
memory, tools/make_goldens.py), and the two inflow/outflow bench shapes (4096 x 16384
two-level, 1024 x 4096 four-level; oracle/inflow.py, R20).  Each golden stores the oracle's Psi coefficients (the
library consumes the same data), the residual history, K, 8 sampled C-rows after every
iteration and 8 sampled rows of the final FULL solution.

Bar (R16/R18): identical K, history within 1e-12 relative plus the R18 floor,
every sampled iterate row within 1e-12 of max|U| relative.
"""
import glob
import json
import math
import os

import numpy as np
import pytest

import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REL = 1e-12
GOLD = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "fullsize_*.npz")))


def _load(path):
    z = np.load(path)
    meta = json.loads(str(z["meta"]))
    L = meta["levels"]
    psi = [{"kind": "stencil", "offsets": [int(o) for o in z[f"psi{l}_offsets"]],
            "coeffs": [float(c) for c in z[f"psi{l}_coeffs"]]} for l in range(L - 1)]
    return meta, psi, z


def _workload(meta):
    base = W.ALL[meta["workload"].split("@")[0]]
    w = base.scaled(meta["nx"], meta["nt"], levels=meta["levels"])
    for k in ("m", "order", "tableau", "cfl", "relax", "u0_kind", "u0_seed", "guess_seed",
              "guess_lo", "tol"):
        assert getattr(w, k) == meta[k], k
    return w


def test_goldens_present():
    names = {os.path.basename(p) for p in GOLD}
    for n in ("fullsize_cfg3_full.npz", "fullsize_cfg4_full.npz",
              "fullsize_cfg5_8192x65536.npz", "fullsize_inflow_erk3_full.npz",
              "fullsize_inflow_erk3_ml_full.npz"):
        assert n in names, n


def compare_with_golden(path, options=None):
    """Run the library on a golden's workload; return (K, hist errors, per-iteration C-row
    errors, final-row error, meta) without asserting."""
    from paper_1910_03726_b200 import binding, problem
    binding.lib()
    meta, psi, z = _load(path)
    w = _workload(meta)
    K = int(z["iterations"])
    ho = np.array(z["history"])
    assert bool(z["converged"]) and len(ho) == K + 1
    s = binding.MGRIT(w.nx, w.nt, w.m, w.alpha, w.cfl, w.order, w.tableau, w.levels, psi,
                      w.relax, options=options)
    if meta.get("boundary", "periodic") == "inflow":   # inflow data: the derivative table (R20)
        stages = s.coefficients()[1].shape[0]
        dg = W.inflow_sin4_derivatives(np.arange(w.nt) * w.dt, w.order + stages)
        s.set_inflow(torch.from_numpy(dg).cuda())
    s.set_cycle(meta["cycle"])
    g = problem.device_guess(w)
    s.set_guess(g)
    out = torch.empty_like(g)
    # max_iter = K: K is identical iff the solve converges at K and not at K-1
    res = s.solve(w.tol, K, out=out, keep_crows=True)
    hg = np.array(res["history"])
    umax = float(z["umax"])
    floor = 1e-15 * math.sqrt(2 * w.nt * w.dt) * umax
    ci = torch.as_tensor(z["crow_idx"], device="cuda")
    crow_err = []
    for k in range(min(K, res["iterations"])):
        got = res["crows"][k].index_select(0, ci).cpu().numpy()
        ref = z["crows"][k]
        crow_err.append(float(np.max(np.abs(got - ref)) / np.max(np.abs(ref))))
    fi = torch.as_tensor(z["final_idx"], device="cuda")
    got = out.index_select(0, fi).cpu().numpy()
    final_err = float(np.max(np.abs(got - z["final_rows"])) / umax)
    hist_ok = [abs(a - b) <= REL * abs(b) + floor for a, b in zip(hg, ho)]
    return dict(K=K, res=res, hg=hg, ho=ho, hist_ok=hist_ok, crow_err=crow_err,
                final_err=final_err, meta=meta, w=w)


@pytest.mark.parametrize("path", GOLD, ids=lambda p: os.path.basename(p)[9:-4])
def test_fullsize_solve_vs_oracle_golden(path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = compare_with_golden(path)
    K, res, hg, ho = r["K"], r["res"], r["hg"], r["ho"]
    herr = np.abs(hg - ho[: len(hg)]) / np.abs(ho[: len(hg)])
    print(f"\n[golden {r['meta']['name']}] K={K} hist rel.err max {herr.max():.2e}; C-row rel.err "
          f"per iteration {['%.1e' % e for e in r['crow_err']]}; final rows {r['final_err']:.2e}")
    # max_iter = K: K is identical iff the solve converges at K and not at K-1
    assert res["iterations"] == K and res["converged"], (res["iterations"], hg)
    assert hg[K - 1] >= r["w"].tol
    assert all(r["hist_ok"]), list(zip(hg, ho))
    assert max(r["crow_err"]) <= REL, r["crow_err"]
    assert r["final_err"] <= REL, r["final_err"]

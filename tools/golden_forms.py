"""A/B of the explicit step's algebraic form against the full-size oracle goldens
(R5): per-iteration C-row errors for each step form of option stage_form
(1 plain stage form, 2 folded last stage, 3 Shu-Osher exact-operator, 4 incremental)."""
import glob
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from test_gpu_fullsize_goldens import compare_with_golden  # noqa: E402

names = sys.argv[1:] or ["cfg5_8192x65536", "cfg5_fcycle_1024x16384", "cfg3_full"]
for n in names:
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_{n}.npz")
    for form in [int(f) for f in os.environ.get("FORMS", "1 2 3 4").split()]:
        r = compare_with_golden(path, options={"stage_form": (form,)})
        print(f"{n} stage_form={form} K={r['res']['iterations']}/{r['K']} crow_err="
              f"{['%.2e' % e for e in r['crow_err']]} final={r['final_err']:.2e} "
              f"hist_ok={all(r['hist_ok'])}", flush=True)

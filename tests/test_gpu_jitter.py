"""Race stress of the asynchronous kernels (compute-sanitizer is closed on this GPU pool:
profiles/r02_sanitizer_closed.log).

libmgrit_jitter.so is the same source built with -DMG_JITTER: every mbarrier wait, bulk
copy / reduce-add issue, DSMEM st.async, named barrier, cp.async wait and CTA edge
exchange first sleeps a pseudo-random 0..2 us (uniform per warp, seeded by the clock), so
the CTAs of a cluster, the producer and compute warps, the warps of a CTA and the copy
engine interleave differently on every run.  A result that depends on the interleaving --
a missing wait, a ring slot or receive buffer reused too early, a WAR hazard the
"causality" argument of the cluster kernels (coarse.cu) does not cover -- then changes.
Each case must give, over several jittered runs, the production build's residual history
and bit-identical FULL solution and C-rows.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = ["tiles_vcycle", "cluster_tb", "cluster_ca", "cluster_plain", "seq_periodic",
         "whole_rows", "sdirk", "rk_coarse_ideal", "rk_coarse_redisc", "cfg2", "cfg4",
         "cfg3_ca", "cfg5_fullwidth", "two_level_16384", "cfg3", "inflow_two_level",
         "cfg4_overlap16"]
RUNS = 3


def _run(case, jitter):
    env = dict(os.environ)
    if jitter:
        env["MGRIT_LIBRARY"] = "jitter"
    else:
        env.pop("MGRIT_LIBRARY", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "jitter_run.py"), case],
                       capture_output=True, text=True, env=env, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def jitter_lib():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_03726_b200 import build
    return build.build(variant="jitter")      # compiled once (minutes) if missing


@pytest.mark.parametrize("case", CASES)
def test_jittered_runs_bitwise_equal(case, jitter_lib):
    ref = _run(case, False)
    assert ref["lib"] == "libmgrit.so"
    for r in range(RUNS):
        got = _run(case, True)
        assert got["lib"] == "libmgrit_jitter.so"
        assert got["iterations"] == ref["iterations"], (r, got, ref)
        assert got["history"] == ref["history"], (r, got["history"], ref["history"])
        assert got["out_sha256"] == ref["out_sha256"], (r, case)
        assert got["crows_sha256"] == ref["crows_sha256"], (r, case)

"""Build libmgrit.so (hand-written sm_100a CUDA + C ABI) in-tree with nvcc."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmgrit.so")
# race-stress variant (tma.cuh / device.cuh mg_jitter): random sleeps at every asynchronous
# protocol point; used only by tests/test_gpu_jitter.py
JITTER_LIB = os.path.join(HERE, "libmgrit_jitter.so")
SOURCES = ["mgrit_api.cu", "sweep.cu", "coarse.cu", "levels.cu", "graph.cu", "psifit.cu",
           "bounded.cu"]
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def build(verbose: bool = False, force: bool = False, variant: str = "") -> str:
    """variant "" -> libmgrit.so; "jitter" -> libmgrit_jitter.so (-DMG_JITTER)."""
    lib = JITTER_LIB if variant == "jitter" else LIB
    extra = ["-DMG_JITTER"] if variant == "jitter" else []
    tag = "." + variant if variant else ""
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    deps.append(os.path.join(ROOT, "include", "mgrit.h"))
    if not force and os.path.exists(lib):
        lt = os.path.getmtime(lib)
        if all(os.path.getmtime(d) <= lt for d in deps):
            return LIB
    # objects are kept (git-ignored): a translation unit is recompiled only when its source
    # or any header is newer than its object
    hdr_t = max(os.path.getmtime(d) for d in deps[len(srcs):])
    objs = []
    procs = []
    for s in srcs:
        o = os.path.join(CSRC, os.path.basename(s) + tag + ".o")
        objs.append(o)
        if not force and os.path.exists(o) and os.path.getmtime(o) >= max(hdr_t, os.path.getmtime(s)):
            continue
        cmd = [nvcc(), *NVCC_FLAGS, *extra, "-c", s, "-o", o]
        procs.append((cmd, o, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    log = []
    failed = None
    for cmd, o, p in procs:
        out, _ = p.communicate()
        log.append(out)
        with open(o + ".log", "w") as f:
            f.write(out)
        if p.returncode != 0:
            sys.stderr.write(out)
            if os.path.exists(o):
                os.remove(o)
            failed = failed or cmd
    if failed:
        raise RuntimeError("nvcc failed: " + " ".join(failed))
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", lib]
    subprocess.run(cmd, check=True)
    # ptxas report of every unit (the logs of units not recompiled this time are kept)
    log = []
    for o in objs:
        if os.path.exists(o + ".log"):
            log.append(open(o + ".log").read())
    if verbose:
        sys.stdout.write("".join(log))
    with open(os.path.join(HERE, f"ptxas{tag}.log"), "w") as f:
        f.write("".join(log))
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True,
                variant="jitter" if "--jitter" in sys.argv else ""))

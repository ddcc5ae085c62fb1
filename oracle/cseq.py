"""ORACLE / CPU baseline only: ctypes front end of oracle/seqstep.c (plain sequential
time stepping, stage form, OpenMP over space).  Test infrastructure — see
oracle/__init__.py.  The coefficients come from oracle.discretization (same data as the
numpy oracle); the result is bitwise the numpy oracle's `sequential` (pinned in
tests/test_oracle_seqstep.py)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import discretization as D

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "seqstep.c")
LIB = os.path.join(HERE, "libseqstep.so")
_lib = None


def build(force: bool = False) -> str:
    """gcc -O2 -fopenmp -ffp-contract=off (no FMA contraction: numpy's operation order)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                        SRC, "-o", LIB], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.seq_steps.restype = C.c_int
        L.seq_steps.argtypes = [C.c_int, C.c_longlong, C.c_int, C.POINTER(C.c_double),
                                C.POINTER(C.c_double), C.c_int, C.c_int,
                                C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def seq_steps(order: int, tableau: str, cfl: float, u0: np.ndarray, nsteps: int,
              threads: int = 1) -> np.ndarray:
    """Phi^nsteps u0 for an explicit scheme (ERKp + Up), on `threads` host cores."""
    tab = D.tableau(tableau)
    if tab.implicit:
        raise ValueError("seqstep.c covers explicit schemes (the SDIRK oracle solves by DFT)")
    z = D.z_coefficients(order, cfl)
    ds = sorted(z)
    assert ds == list(range(ds[0], ds[-1] + 1))
    zc = np.array([z[d] for d in ds], dtype=np.float64)
    A = np.ascontiguousarray(np.array(tab.A, dtype=np.float64))
    b = np.array(tab.b, dtype=np.float64)
    u = np.array(u0, dtype=np.float64, copy=True)
    st = lib().seq_steps(u.shape[0], nsteps, tab.s, _dp(A), _dp(b), ds[0], len(ds), _dp(zc),
                         _dp(u), threads)
    if st:
        raise RuntimeError("seq_steps failed")
    return u

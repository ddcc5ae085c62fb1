"""Thin ctypes binding of libmgrit.so (include/mgrit.h).  Argument marshalling only:
every step of the MGRIT path runs in the library's sm_100a kernels.  PyTorch provides
device memory (the workspace, the guess, outputs) and the CUDA stream.

The binding fails loudly when the library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmgrit.so")
# MGRIT_LIBRARY=jitter loads the race-stress build (tests/test_gpu_jitter.py only; the same
# ABI, random sleeps at the asynchronous protocol points).  No CPU fallback either way.
if os.environ.get("MGRIT_LIBRARY") == "jitter":
    LIB_PATH = os.path.join(HERE, "libmgrit_jitter.so")
elif os.environ.get("MGRIT_LIBRARY") == "trace":   # -DMG_TRACE build (tools/trace_overlap.sh)
    LIB_PATH = os.path.join(HERE, "libmgrit_trace.so")

TABLEAU = {"erk1": 0, "erk2": 1, "erk3_ssp": 2, "erk3_kutta": 3, "erk4": 4, "erk5": 5,
           "sdirk1": 6, "sdirk2": 7, "sdirk3": 8, "sdirk4": 9}
RELAX = {"F": 0, "C": 1, "FCF": 2}
PSI_KIND = {"stencil": 0, "ideal": 1, "redisc": 2}
STATUS = {0: "OK", -1: "EINVAL", -2: "ENOMEM", -3: "ECUDA", -4: "ENONFINITE", -5: "EUNSUPPORTED",
          -6: "ECOMM"}
OPTION = {"fine_tile": 0, "whole_row": 1, "seq_cluster": 2, "seq_s": 3, "coarse_kernel": 4,
          "seq_cfg": 5, "sdirk_product": 6, "stage_form": 7, "graph": 8, "overlap": 9, "voverlap": 10}
PROF_CLASSES = ("fine_sweep", "level_sweep", "coarse_solve", "interp", "residual", "other")
MAX_LEVELS = 8


class MgritError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class _Psi(C.Structure):
    _fields_ = [("kind", C.c_int), ("nnz", C.c_int), ("offsets", C.POINTER(C.c_int)),
                ("coeffs", C.POINTER(C.c_double)), ("redisc_cfl", C.c_double)]


_lib = None

# (name, restype, argtypes) of every entry point declared in include/mgrit.h
_SIGS = [
    ("mgrit_workspace_bytes", C.c_size_t, [C.c_int, C.c_int, C.c_int, C.c_int]),
    ("mgrit_setup", C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, C.c_double,
                              C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(_Psi), C.c_int,
                              C.c_void_p, C.c_size_t, C.c_void_p]),
    ("mgrit_destroy", None, [C.c_void_p]),
    ("mgrit_last_error", C.c_char_p, [C.c_void_p]),
    ("mgrit_get_coefficients", C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                         C.POINTER(C.c_int), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("mgrit_scheme_coefficients", C.c_int, [C.c_int, C.c_int, C.c_double, C.POINTER(C.c_int),
                                            C.POINTER(C.c_int), C.POINTER(C.c_int),
                                            C.POINTER(C.c_double), C.POINTER(C.c_double),
                                            C.POINTER(C.c_double)]),
    ("mgrit_set_guess", C.c_int, [C.c_void_p, C.c_void_p]),
    ("mgrit_relax", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    ("mgrit_residual", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_double),
                                 C.c_void_p]),
    ("mgrit_coarse_solve", C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    ("mgrit_set_rhs", C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    ("mgrit_set_inflow", C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    ("mgrit_get_forcing", C.c_int, [C.c_void_p, C.c_void_p]),
    ("mgrit_solve", C.c_int, [C.c_void_p, C.c_double, C.c_int, C.c_void_p, C.POINTER(C.c_int),
                              C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_void_p]),
    ("mgrit_set_cycle", C.c_int, [C.c_void_p, C.c_int]),
    ("mgrit_set_final_sweep", C.c_int, [C.c_void_p, C.c_int]),
    ("mgrit_set_option", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.c_int]),
    ("mgrit_overlap_plan", C.c_int, [C.c_longlong, C.c_int, C.POINTER(C.c_int),
                                     C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    ("mgrit_get_crows", C.c_int, [C.c_void_p, C.c_void_p]),
    ("mgrit_fill_guess", C.c_int, [C.c_void_p, C.c_longlong, C.c_longlong, C.c_int,
                                   C.c_uint64, C.c_int, C.c_void_p, C.c_void_p]),
    ("mgrit_workspace_bytes_shard", C.c_size_t, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    ("mgrit_setup_shard", C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, C.c_double,
                                    C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(_Psi),
                                    C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_size_t, C.c_void_p]),
    ("mgrit_solve_shard", C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_void_p,
                                    C.POINTER(C.c_int), C.POINTER(C.c_double),
                                    C.POINTER(C.c_int)]),
    ("mgrit_psi_fit_workspace_bytes", C.c_size_t, [C.c_int]),
    ("mgrit_psi_fit", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                C.POINTER(C.c_int), C.c_double, C.POINTER(C.c_int),
                                C.POINTER(C.c_int), C.POINTER(C.c_double),
                                C.POINTER(C.c_double), C.c_void_p, C.c_size_t, C.c_void_p]),
    ("mgrit_psi_fit_nl_workspace_bytes", C.c_size_t, [C.c_int]),
    ("mgrit_psi_fit_nl", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_int), C.POINTER(C.c_double), C.c_int,
                                   C.POINTER(C.c_int), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.c_void_p, C.c_size_t, C.c_void_p]),
    ("mgrit_profile_enable", C.c_int, [C.c_void_p, C.c_int]),
    ("mgrit_profile_read", C.c_int, [C.c_void_p, C.POINTER(C.c_longlong),
                                     C.POINTER(C.c_double)]),
    ("mgrit_launch_count", C.c_longlong, [C.c_void_p]),
    ("mgrit_describe", C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t]),
]


def lib():
    """Load libmgrit.so (built by paper_1910_03726_b200/build.py); raise if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1910_03726_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in _SIGS:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols() -> List[str]:
    return [s[0] for s in _SIGS]


def _dptr(t) -> Optional[int]:
    if t is None:
        return None
    import torch
    assert isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 \
        and t.is_contiguous(), "expected a contiguous CUDA float64 tensor"
    return t.data_ptr()


def scheme_coefficients(order: int, tableau: str, cfl: float):
    """Host-only: the library's z_d (d = z_lo..) and Butcher (A, b)."""
    s, zlo, zn = C.c_int(), C.c_int(), C.c_int()
    z = (C.c_double * 8)()
    A = (C.c_double * 36)()
    b = (C.c_double * 6)()
    st = lib().mgrit_scheme_coefficients(order, TABLEAU[tableau], cfl, C.byref(s), C.byref(zlo),
                                         C.byref(zn), z, A, b)
    if st:
        raise MgritError(st, "mgrit_scheme_coefficients")
    S = s.value
    zd = {zlo.value + k: z[k] for k in range(zn.value)}
    Am = np.array(A[:]).reshape(6, 6)[:S, :S].copy()
    return zd, Am, np.array(b[:S])


def psi_fit_device(order: int, tableau: str, cfl: float, nx: int, m: int, levels: int,
                   widths: Sequence[int] = (), eta: Optional[float] = None, stream=None):
    """mgrit_psi_fit: the Psi hierarchy fitted on the GPU (include/mgrit.h).  Returns
    library inputs [{"kind": "stencil", "offsets", "coeffs", "imag"}, ...]."""
    import torch
    L = lib()
    nb = L.mgrit_psi_fit_workspace_bytes(nx)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    nl = levels - 1
    T = 64
    offs = (C.c_int * (nl * T))()
    nnz = (C.c_int * nl)()
    cof = (C.c_double * (nl * T))()
    imag = (C.c_double * nl)()
    wid = (C.c_int * max(1, nl))(*[int(v) for v in list(widths)[:nl]]) if widths else None
    st = L.mgrit_psi_fit(nx, order, TABLEAU[tableau], cfl, m, levels, wid,
                         float(eta) if eta else 0.0, offs, nnz, cof, imag, ws.data_ptr(), nb,
                         C.c_void_p(_stream(stream)))
    if st:
        raise MgritError(st, "mgrit_psi_fit")
    out = []
    for l in range(nl):
        n = nnz[l]
        out.append({"kind": "stencil", "offsets": [offs[l * T + a] for a in range(n)],
                    "coeffs": [cof[l * T + a] for a in range(n)], "imag": imag[l]})
    return out


def psi_fit_nl_device(order: int, tableau: str, cfl: float, nx: int, m: int, nt: int,
                      offsets: Sequence[int], coeffs: Sequence[float], max_iter: int = 30,
                      stream=None):
    """mgrit_psi_fit_nl: the nonlinear least-squares Psi of PAPER.md Appendix B on the GPU, by
    Levenberg-Marquardt from `coeffs` (the linear fit).  Returns a library input dict with
    "objective", "iterations" and the objective "history"."""
    import torch
    L = lib()
    nb = L.mgrit_psi_fit_nl_workspace_bytes(nx)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    n = len(offsets)
    offs = (C.c_int * n)(*[int(d) for d in offsets])
    cof = (C.c_double * n)(*[float(v) for v in coeffs])
    its = C.c_int()
    obj = C.c_double()
    hist = (C.c_double * (max_iter + 1))()
    st = L.mgrit_psi_fit_nl(nx, order, TABLEAU[tableau], cfl, m, nt, n, offs, cof, max_iter,
                            C.byref(its), C.byref(obj), hist, ws.data_ptr(), nb,
                            C.c_void_p(_stream(stream)))
    if st:
        raise MgritError(st, "mgrit_psi_fit_nl")
    return {"kind": "stencil", "offsets": list(offsets), "coeffs": [cof[a] for a in range(n)],
            "objective": obj.value, "iterations": its.value,
            "history": [hist[i] for i in range(its.value + 1)]}


def overlap_plan(nc: int, want: int):
    """mgrit_overlap_plan: (C, [(j0, j1), ...]) of the overlapped two-level iteration (host-only)."""
    ch = C.c_int()
    n = max(1, want)
    j0 = (C.c_longlong * n)()
    j1 = (C.c_longlong * n)()
    st = lib().mgrit_overlap_plan(nc, want, C.byref(ch), j0, j1)
    if st:
        raise MgritError(st, "mgrit_overlap_plan")
    return ch.value, [(j0[i], j1[i]) for i in range(ch.value)]


def fill_guess(dst, seed: int, lo: float = -1.0, u0=None, row0: int = 0, stream=None):
    """Fill a (rows, nx) CUDA float64 tensor with the counter-based guess (R4)."""
    import torch
    rows, nx = dst.shape
    st = lib().mgrit_fill_guess(_dptr(dst), row0, rows, nx, seed, 0 if lo == -1.0 else 1,
                                _dptr(u0), C.c_void_p(_stream(stream)))
    if st:
        raise MgritError(st, "mgrit_fill_guess")
    return dst


def psi_array(psi: Sequence[Dict], levels: int):
    """The mgrit_psi array of levels-1 coarse operators (+ the ctypes buffers to keep)."""
    arr = (_Psi * max(1, levels - 1))()
    keep = []
    for l, p in enumerate(psi):
        kind = PSI_KIND[p["kind"]]
        arr[l].kind = kind
        if kind == 0:
            offs = (C.c_int * len(p["offsets"]))(*[int(o) for o in p["offsets"]])
            cof = (C.c_double * len(p["coeffs"]))(*[float(c) for c in p["coeffs"]])
            keep += [offs, cof]
            arr[l].nnz = len(p["offsets"])
            arr[l].offsets = C.cast(offs, C.POINTER(C.c_int))
            arr[l].coeffs = C.cast(cof, C.POINTER(C.c_double))
        arr[l].redisc_cfl = float(p.get("cfl", 0.0))
    return arr, keep


def _stream(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class MGRIT:
    """One problem (nx, nt, m, scheme, Psi hierarchy) bound to a CUDA stream.

    psi: list of levels-1 dicts: {"kind": "stencil", "offsets": [...], "coeffs": [...]},
    {"kind": "ideal"} or {"kind": "redisc", "cfl": c'}.
    """

    def __init__(self, nx: int, nt: int, m: int, alpha: float, cfl: float, order: int,
                 tableau: str, levels: int, psi: Sequence[Dict], relax: str = "FCF",
                 stream=None, device: str = "cuda", options: Optional[Dict] = None):
        import torch
        self.nx, self.nt, self.m, self.levels = nx, nt, m, levels
        self.alpha, self.cfl, self.order, self.tableau = alpha, cfl, order, tableau
        self.relax = relax
        self.dx = 2.0 / nx
        self.dt = cfl * self.dx / alpha
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        nbytes = lib().mgrit_workspace_bytes(nx, nt, m, levels)
        if nbytes == 0:
            raise MgritError(-1, f"invalid sizes nx={nx} nt={nt} m={m} levels={levels}")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=device)
        arr, self._keep = psi_array(psi, levels)
        ctx = C.c_void_p()
        st = lib().mgrit_setup(C.byref(ctx), nx, nt, m, alpha, cfl, order, TABLEAU[tableau],
                               levels, arr, RELAX[relax], self.workspace.data_ptr(), nbytes,
                               C.c_void_p(self.stream.cuda_stream))
        if st:
            raise MgritError(st, "mgrit_setup failed (see stderr)")
        self.ctx = ctx
        self.guess = None
        for k, v in (options or {}).items():
            self.set_option(k, v)

    def __del__(self):
        try:
            if getattr(self, "ctx", None):
                lib().mgrit_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass

    def _check(self, st, what):
        if st:
            msg = lib().mgrit_last_error(self.ctx)
            raise MgritError(st, f"{what}: {msg.decode() if msg else ''}")

    # ---- FULL-state primitives (level 0: fine grid; level l >= 1: Psi_l with RHS g_l) ----
    def relax_full(self, U, kind: str = "FCF", level: int = 0):
        self._check(lib().mgrit_relax(self.ctx, level, RELAX[kind], _dptr(U)), "mgrit_relax")

    def residual_full(self, U, want_r: bool = False, level: int = 0):
        import torch
        norm = C.c_double()
        ntl = self.nt // self.m ** level
        r = torch.empty((ntl // self.m + 1, self.nx), dtype=torch.float64,
                        device=U.device) if want_r else None
        self._check(lib().mgrit_residual(self.ctx, level, _dptr(U), C.byref(norm), _dptr(r)),
                    "mgrit_residual")
        return (norm.value, r) if want_r else norm.value

    def coarse_solve_full(self, U, level: int = 0):
        self._check(lib().mgrit_coarse_solve(self.ctx, level, _dptr(U)), "mgrit_coarse_solve")

    def set_rhs(self, level: int, g=None):
        """mgrit_set_rhs: the level-l right-hand side g_l of the level primitives (None: 0)."""
        self._rhs_keep = getattr(self, "_rhs_keep", {})
        self._rhs_keep[level] = g
        self._check(lib().mgrit_set_rhs(self.ctx, level, _dptr(g)), "mgrit_set_rhs")

    def set_inflow(self, dg=None, enable: bool = True):
        """mgrit_set_inflow: inflow/outflow boundaries (PAPER.md 4.5); dg = nt x (order + s)
        device array of inflow derivatives g^(r)(t_n) (None: homogeneous inflow)."""
        if dg is not None:
            assert dg.is_cuda and dg.dtype.is_floating_point and dg.is_contiguous()
            assert dg.shape[0] == self.nt
        self._check(lib().mgrit_set_inflow(self.ctx, 1 if enable else 0, _dptr(dg)),
                    "mgrit_set_inflow")

    def get_forcing(self):
        """mgrit_get_forcing: the nt x 24 compact forcing rows b_n (device tensor)."""
        import torch
        out = torch.empty((self.nt, 24), dtype=torch.float64, device=self.workspace.device)
        self._check(lib().mgrit_get_forcing(self.ctx, _dptr(out)), "mgrit_get_forcing")
        return out

    # ---- production solve -------------------------------------------------------
    def set_guess(self, guess):
        assert tuple(guess.shape) == (self.nt + 1, self.nx)
        self.guess = guess
        self._check(lib().mgrit_set_guess(self.ctx, _dptr(guess)), "mgrit_set_guess")

    def set_cycle(self, cycle: str):
        """Multilevel cycle of `solve`: "V" (default) or "F" (R19)."""
        self._check(lib().mgrit_set_cycle(self.ctx, {"V": 0, "F": 1}[cycle]), "mgrit_set_cycle")

    def set_option(self, name: str, values: Sequence[int] = ()):
        """mgrit_set_option (include/mgrit.h): a kernel-configuration override, () = default."""
        vals = [int(v) for v in values]
        arr = (C.c_int * max(1, len(vals)))(*vals)
        self._check(lib().mgrit_set_option(self.ctx, OPTION[name], arr, len(vals)),
                    f"mgrit_set_option({name})")

    def set_final_sweep(self, mode: str):
        """mgrit_set_final_sweep: "off", "predict" (default) or "always" (include/mgrit.h)."""
        self._check(lib().mgrit_set_final_sweep(self.ctx, {"off": 0, "predict": 1, "always": 2}[mode]),
                    "mgrit_set_final_sweep")

    def solve(self, tol: float = 1e-10, max_iter: int = 64, out=None, keep_crows: bool = False):
        import torch
        iters, conv = C.c_int(), C.c_int()
        hist = (C.c_double * (max_iter + 1))()
        crows = None
        if keep_crows:
            crows = torch.empty((max(1, max_iter), self.nt // self.m + 1, self.nx),
                                dtype=torch.float64, device=self.guess.device)
        st = lib().mgrit_solve(self.ctx, tol, max_iter, _dptr(out), C.byref(iters), hist,
                               C.byref(conv), _dptr(crows))
        k = iters.value
        res = {"iterations": k, "history": list(hist[:k + 1]), "converged": bool(conv.value),
               "status": st}
        if keep_crows:
            res["crows"] = crows[:k]
        if st and st != -4:
            self._check(st, "mgrit_solve")
        return res

    def crows(self):
        import torch
        out = torch.empty((self.nt // self.m + 1, self.nx), dtype=torch.float64,
                          device=self.guess.device)
        self._check(lib().mgrit_get_crows(self.ctx, _dptr(out)), "mgrit_get_crows")
        return out

    def coefficients(self):
        s, zlo, zn = C.c_int(), C.c_int(), C.c_int()
        z = (C.c_double * 8)()
        A = (C.c_double * 36)()
        b = (C.c_double * 6)()
        self._check(lib().mgrit_get_coefficients(self.ctx, C.byref(s), C.byref(zlo), C.byref(zn),
                                                 z, A, b), "coefficients")
        S = s.value
        return ({zlo.value + k: z[k] for k in range(zn.value)},
                np.array(A[:]).reshape(6, 6)[:S, :S].copy(), np.array(b[:S]))

    # ---- profiling --------------------------------------------------------------
    def profile(self, on: bool = True):
        self._check(lib().mgrit_profile_enable(self.ctx, 1 if on else 0), "profile_enable")

    def profile_read(self):
        n = (C.c_longlong * 6)()
        ms = (C.c_double * 6)()
        self._check(lib().mgrit_profile_read(self.ctx, n, ms), "profile_read")
        return {k: (n[i], ms[i]) for i, k in enumerate(PROF_CLASSES)}

    def launch_count(self) -> int:
        return lib().mgrit_launch_count(self.ctx)

    def describe(self) -> str:
        buf = C.create_string_buffer(256)
        self._check(lib().mgrit_describe(self.ctx, buf, 256), "describe")
        return buf.value.decode()

"""Bind a BASELINE.json workload (workloads/) to the library: Psi inputs, solver, guess."""
from __future__ import annotations

from typing import Dict, List, Optional

import numpy as np

from . import binding, psi as psimod


def psi_inputs(w, device: bool = False, nonlinear: bool = False) -> List[Dict]:
    """Coarse operators of a workload as library inputs (LSQ fit): host numpy
    (default) or on the GPU (mgrit_psi_fit, device=True); nonlinear=True (two-level, explicit
    schemes, device only) refines the linear fit by the nonlinear least squares of PAPER.md
    Appendix B (mgrit_psi_fit_nl)."""
    if w.psi_kind == "ideal":
        return [{"kind": "ideal"}]
    if w.psi_kind == "redisc":
        return [{"kind": "redisc", "cfl": w.redisc_cfl}]
    if nonlinear and not (device and w.levels == 2):
        raise ValueError("the nonlinear fit is two-level and runs on the device")
    if device:
        out = binding.psi_fit_device(w.order, w.tableau, w.cfl, w.nx, w.m, w.levels,
                                     w.psi_widths, w.psi_eta)
        for lvl, p in enumerate(out):
            if p["imag"] > psimod.IMAG_TOL:
                raise psimod.PsiRejected(f"level {lvl + 2}: imaginary component {p['imag']:.2e}")
        if nonlinear:
            out = [binding.psi_fit_nl_device(w.order, w.tableau, w.cfl, w.nx, w.m, w.nt,
                                             out[0]["offsets"], out[0]["coeffs"])]
        return out
    return psimod.hierarchy(w.order, w.tableau, w.cfl, w.nx, w.m, w.levels,
                            w.psi_widths, w.psi_eta)


def make_solver(w, psi: Optional[List[Dict]] = None, stream=None,
                options: Optional[Dict] = None) -> binding.MGRIT:
    s = binding.MGRIT(w.nx, w.nt, w.m, w.alpha, w.cfl, w.order, w.tableau, w.levels,
                      psi if psi is not None else psi_inputs(w), w.relax, stream=stream,
                      options=options)
    if getattr(w, "boundary", "periodic") == "inflow":   # PAPER.md 4.5: u(-1, t) = sin^4(pi t)
        import torch
        import workloads as W
        stages = s.coefficients()[1].shape[0]
        dg = W.inflow_sin4_derivatives(np.arange(w.nt) * w.dt, w.order + stages)
        s.set_inflow(torch.from_numpy(dg).to(s.workspace.device))
    return s


def device_guess(w, device="cuda"):
    """The workload's initial iterate generated on the device (R4)."""
    import torch
    u0 = torch.from_numpy(w.u0()).to(device)
    g = torch.empty((w.nt + 1, w.nx), dtype=torch.float64, device=device)
    binding.fill_guess(g, w.guess_seed, w.guess_lo, u0=u0)
    return g


def dof_updates(w, iterations: int) -> int:
    """Fine space-time DOF updates of a solve: 2*nt*nx per FCF iteration,
    nt*nx per F iteration."""
    per = 2 if w.relax == "FCF" else 1
    return per * w.nt * w.nx * iterations

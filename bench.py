#!/usr/bin/env python
"""bench.py — MGRIT time-to-residual 1e-10 and fine space-time DOF updates/s on B200.

Workload (default): BASELINE.json configs[4] ("cfg5", the throughput run): periodic
advection, nx = 16384, nt = 65536 (8 GiB space-time state), ERK3(SSP)+U3, c = 0.85,
multilevel V-cycle, m = 4, 6 levels, FCF, Psi_l fitted on the host.

A step = one complete MGRIT solve from the (read-only, HBM-resident) initial iterate to
||r|| < 1e-10, including the all-row initial residual and the F-point materialisation of
the full solution.  value = fine DOF updates / s = 2*nt*nx*K / t_step.

--impl reference runs the oracle (numpy, fp64, host cores) on a bounded sample of the
same workload and reports the same metric.

Multi-GPU: the hot path is not sharded (DESIGN.md §7 "replicas only"): each rank solves
its own replica; value = all ranks' DOF updates / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "fine space-time DOF updates/s (fp64) & MGRIT time-to-residual 1e-10"
UNIT = "DOF-updates/s"
FP64_PEAK_TFLOPS = 2 * 64 * 148 * 1.965e9 / 1e12   # 64 DFMA/clk/SM x 148 SMs x 1965 MHz


def _measured_fp64_peak():
    """Median sustained DFMA rate of tools/probe_fp64 (tools/probe_fp64.sh), with the SM clock
    nvidia-smi recorded during that run (profiles/r02_fp64_probe.json)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r02_fp64_probe.json")))
        return float(d["dfma_tflops_median"]), d.get("sm_mhz_median_under_load")
    except Exception:
        return None, None


# Algorithmic flops per point and step of the stage form: Z with t taps =
# 1 MUL + (t-1) FMA; every nonzero a_il, b_i = 1 FMA (2 flops).  SDIRK3+U3: SURVEY 8(d)'s
# 3 x [banded stage solve ~7 + Z 7] + combinations (2 + 4) + update 6 = 55.
FLOPS_PER_POINT_STEP = {"erk1": 5.0, "erk2": 14.0, "erk3_ssp": 33.0, "erk3_kutta": 33.0,
                        "erk4": 44.0, "erk5": 102.0, "sdirk3": 55.0}
# Flops the kernels actually execute per point-step (last stage folded into
# the update; SSP-RK3 in the Shu-Osher form = 13 DFMA + 1 DADD + 1 DMUL): the FP64-pipe
# view of the same launch, reported beside the algorithmic fraction.
EXEC_FLOPS_PER_POINT_STEP = {"erk1": 4.0, "erk3_ssp": 28.0, "erk3_kutta": 32.0, "erk5": 101.0}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        import torch.distributed as dist
        import torch
        if not dist.is_initialized():
            dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
        return dist, dist.get_rank(), ws
    return None, 0, 1


def _clock_sampler(path):
    q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    try:
        return subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                 "-lms", "200"], stdout=open(path, "w"), stderr=subprocess.DEVNULL)
    except Exception:
        return None


def _clock_summary(path, gpu_index):
    sm, mx, reasons = [], None, set()
    try:
        for line in open(path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or f[0] != str(gpu_index):
                continue
            sm.append(float(f[1]))
            mx = float(f[2])
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
    except Exception:
        pass
    if not sm:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
    return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
            "samples": len(sm)}


def _profile_traffic():
    """dram bytes per fine-sweep launch from the committed ncu summary, if present."""
    p = os.path.join(ROOT, "profiles", "fine_sweep_ncu.json")
    try:
        d = json.load(open(p))
        return (d[0] if isinstance(d, list) else d).get("dram_bytes_per_launch")
    except Exception:
        return None


def aggregate(ms_local: float, dof_local: int, dist=None):
    """Replicas: every rank solves its own replica; the job time is the
    max over ranks (device-timed), the value all ranks' DOF updates / that time."""
    world = 1
    ms = ms_local
    dof = dof_local
    if dist is not None and dist.is_initialized():
        import torch
        world = dist.get_world_size()
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([ms_local, float(dof_local)], dtype=torch.float64, device=dev)
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        ms = float(tmax[0].item())
        dof = int(t[1].item())
    return ms, dof / (ms / 1e3), world


# ------------------------------------------------------------------ oracle sample
def host_info():
    """CPU model and logical core count of the host the CPU baselines ran on."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu": model, "nproc": os.cpu_count()}


def oracle_sample(w, budget_s: float = 12.0):
    """The oracle, as it stands, on a bounded sample of the workload: full-width rows
    (nx as configured), nt reduced so one V-cycle iteration takes ~budget_s."""
    from oracle import discretization as D, mgrit as M, psi as OP
    nt_s = 64 * w.m ** 2
    levels = 3
    ws = w.scaled(w.nx, nt_s, levels=levels)
    phi = D.make_phi(ws.order, ws.tableau, ws.cfl, ws.nx)
    fits = OP.fit_hierarchy(phi, ws.nx, ws.m, ws.cfl, ws.psi_widths[: levels - 1])
    phis = [phi] + [D.StencilPhi(f.stencil, ws.nx) for f in fits]
    U = ws.guess()
    t0 = time.perf_counter()
    iters = 0
    while True:
        M.vcycle(0, U, None, phis, ws.m, ws.relax)
        M.residual_norm(U, phi, ws.dx, ws.dt)
        iters += 1
        if time.perf_counter() - t0 > budget_s or iters >= 8:
            break
    dt = time.perf_counter() - t0
    dof = 2 * nt_s * ws.nx * iters
    return {"value": dof / dt, "unit": UNIT, "cores": 1, "kind": "oracle", "host": host_info(),
            "sample": f"{iters} oracle V-cycle iteration(s) (FCF, m={ws.m}, {levels} levels) on "
                      f"nx={ws.nx} x nt={nt_s} rows of the {w.name} recipe, numpy fp64, "
                      f"{dt:.1f} s"}


def sequential_sample(w, budget_s: float = 6.0):
    """Plain sequential time-stepping, the paper's serial baseline,
    on the host: oracle/seqstep.c (stage form, bitwise the numpy oracle's `sequential`,
    OpenMP over space).  All host cores run the FULL workload (nt steps); one core runs a
    bounded sample of the steps (its full-run time is extrapolated and labelled so)."""
    from oracle import cseq
    if D_tab_implicit(w):
        return None
    ncores = os.cpu_count() or 1
    u = w.u0()
    t0 = time.perf_counter()
    cseq.seq_steps(w.order, w.tableau, w.cfl, u, w.nt, threads=ncores)
    t_all = time.perf_counter() - t0
    n1 = 256
    t0 = time.perf_counter()
    while True:
        cseq.seq_steps(w.order, w.tableau, w.cfl, u, n1, threads=1)
        dt1 = time.perf_counter() - t0
        if dt1 > budget_s / 4 or n1 >= w.nt:
            break
        n1 *= 2
        t0 = time.perf_counter()
    rate1 = n1 * w.nx / dt1
    return {"value": w.nt * w.nx / t_all, "unit": UNIT, "cores": ncores, "threads": ncores,
            "kind": "sequential time-stepping (oracle/seqstep.c, OpenMP over space)",
            "host": host_info(), "time_s": round(t_all, 3),
            "sample": f"full run: all {w.nt} steps of {w.tableau}+U{w.order} at nx={w.nx}, "
                      f"fp64 stage form, {ncores} threads",
            "single_core": {"value": rate1, "unit": UNIT, "cores": 1,
                            "sample": f"{n1} of {w.nt} steps on 1 thread, {dt1:.2f} s",
                            "full_run_s_extrapolated": round(w.nt * w.nx / rate1, 1)}}


def D_tab_implicit(w):
    from oracle import discretization as D
    return D.tableau(w.tableau).implicit


# ------------------------------------------------------------------ our arm
def run_ours(args, w):
    import torch
    from paper_1910_03726_b200 import binding, problem
    from paper_1910_03726_b200 import build as B

    dist, rank, world = _dist()
    B.build()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    psi = problem.psi_inputs(w)
    opts = {k: tuple(int(x) for x in v.split(",")) for k, v in (o.split("=") for o in args.opt)}
    s = problem.make_solver(w, psi, stream=stream, options=opts)
    s.set_cycle(args.cycle)
    s.set_final_sweep(args.final_sweep)
    guess = problem.device_guess(w)
    out = torch.empty_like(guess)
    s.set_guess(guess)
    torch.cuda.synchronize()

    def step():
        return s.solve(w.tol, w.max_iter, out=out)

    for _ in range(args.warmup):
        res = step()
    # ---- timed region: K complete solves, CUDA events on the solver's stream ----
    clk_path = os.path.join(ROOT, "gpurun_out", f"bench_clocks_r{rank}.csv")
    os.makedirs(os.path.dirname(clk_path), exist_ok=True)
    sampler = _clock_sampler(clk_path) if rank == 0 else None
    time.sleep(0.3 if sampler else 0)
    def timed(profiled: bool):
        """K solves bracketed by a barrier + synchronize; per-launch CUDA events on the
        solver's stream when `profiled` (they add ~1.5 % to a solve)."""
        s.profile(profiled)                      # also resets the launch counter
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        its = []
        r = None
        for _ in range(args.steps):
            r = step()
            its.append(r["iterations"])
        e1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t = e0.elapsed_time(e1)
        pr = s.profile_read()
        nl = s.launch_count()
        s.profile(False)
        return t, its, pr, nl, r

    # headline: the K solves without instrumentation; then the same K solves again with
    # per-launch events for the roofline and the kernel-time shares
    ms_total, iters, _, launches, res = timed(False)
    ms_total_prof, iters_p, prof, _, _ = timed(not args.no_prof)
    iters += iters_p
    if sampler:
        sampler.terminate()
        sampler.wait()
    K = iters[-1]
    assert all(k == K for k in iters), iters
    dof = problem.dof_updates(w, K)
    ms, value, world = aggregate(ms_total / args.steps, dof, dist)

    # ---- roofline of the dominant kernel: the fine FCF sweep (class fine_sweep) ----
    n_f, ms_f = prof["fine_sweep"]
    nc = w.nt // w.m
    point_steps = w.nx * (nc * w.m + (nc - 1) * w.m)          # phase 1 + phase 2
    flops = FLOPS_PER_POINT_STEP[w.tableau] * point_steps
    avg_ms = ms_f / max(n_f, 1)
    achieved = flops / (avg_ms / 1e3) / 1e12 if avg_ms > 0 else 0.0  # 0: --no-prof
    probe_tf, probe_mhz = _measured_fp64_peak()
    ex = EXEC_FLOPS_PER_POINT_STEP.get(w.tableau)
    executed = None
    if ex and avg_ms > 0:
        a_ex = ex * point_steps / (avg_ms / 1e3) / 1e12
        executed = {"flops_per_point_step": ex, "achieved": round(a_ex, 3),
                    "frac": round(a_ex / FP64_PEAK_TFLOPS, 4),
                    "frac_vs_probe": round(a_ex / probe_tf, 4) if probe_tf else None}
    shares = {k: round(v[1] / max(ms_total_prof, 1e-9), 4) for k, v in prof.items()}
    # ---- sequential coarse solve: ns per coarse step vs its FP64 floor ----
    desc = s.describe()
    n_c, ms_c = prof["coarse_solve"]
    nsteps_c = w.nt // (w.m ** (w.levels - 1))
    coarse = {"kernel": desc.split("coarse=")[-1], "launches": n_c,
              "steps_per_launch": nsteps_c,
              "ns_per_step": round(ms_c / max(n_c, 1) / nsteps_c * 1e6, 1) if n_c else None}
    if w.psi_kind == "stencil" and n_c:
        ops = psi[-1]
        nu = ops["offsets"][-1] - ops["offsets"][0] + 1
        cl = 1
        if "CL=" in desc:
            cl = int(desc.split("CL=")[1].split(",")[0].split(">")[0])
        elif "tiles=" in coarse["kernel"]:
            cl = min(148, int(coarse["kernel"].split("tiles=")[1].split()[0]))
        floor = nu * w.nx * 2 / (cl * FP64_PEAK_TFLOPS * 1e12 / 148) * 1e9
        coarse.update({"taps": nu, "sms": cl, "fp64_floor_ns_per_step": round(floor, 1)})

    # ---- end to end through the public API with host buffers -----------------------
    e2e = None
    if not args.no_e2e:
        u0_host = torch.from_numpy(w.u0()).pin_memory()
        out_host = torch.empty((w.nt + 1, w.nx), dtype=torch.float64).pin_memory()
        u0_dev = torch.empty_like(u0_host, device="cuda")
        tt = []
        for it in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            u0_dev.copy_(u0_host, non_blocking=True)
            binding.fill_guess(guess, w.guess_seed, w.guess_lo, u0=u0_dev, stream=stream)
            r = step()
            out_host.copy_(out, non_blocking=True)
            a1.record(stream)
            torch.cuda.synchronize()
            if it >= args.warmup:
                tt.append(a0.elapsed_time(a1))
        ms_e2e = sum(tt) / len(tt)
        e2e = {"value": dof * world / (ms_e2e / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(u0_host.numel() * 8),
               "d2h_bytes_per_step": int(out_host.numel() * 8),
               "ms_per_step": round(ms_e2e, 3),
               "note": "H2D u0 (pinned), device-generated random iterate (R4), solve, "
                       "D2H of the full (nt+1) x nx solution"}
        if world == 1:
            # the same with the initial iterate uploaded from pinned host memory as well
            # (the whole (nt+1) x nx guess, not just u0, crosses PCIe every step)
            binding.fill_guess(guess, w.guess_seed, w.guess_lo, u0=u0_dev, stream=stream)
            guess_host = torch.empty((w.nt + 1, w.nx), dtype=torch.float64).pin_memory()
            guess_host.copy_(guess)
            torch.cuda.synchronize()
            th = []
            for it in range(args.warmup + args.steps):
                torch.cuda.synchronize()
                a0 = torch.cuda.Event(enable_timing=True)
                a1 = torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                guess.copy_(guess_host, non_blocking=True)
                step()
                out_host.copy_(out, non_blocking=True)
                a1.record(stream)
                torch.cuda.synchronize()
                if it >= args.warmup:
                    th.append(a0.elapsed_time(a1))
            ms_h = sum(th) / len(th)
            e2e["host_guess"] = {"value": dof / (ms_h / 1e3), "unit": UNIT,
                                 "h2d_bytes_per_step": int(guess_host.numel() * 8),
                                 "d2h_bytes_per_step": int(out_host.numel() * 8),
                                 "ms_per_step": round(ms_h, 3),
                                 "note": "H2D of the whole initial iterate (pinned), solve, "
                                         "D2H of the full solution"}
            del guess_host
        del out_host

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "nx": w.nx, "nt": w.nt, "scheme": f"{w.tableau}+U{w.order}",
                   "cfl": w.cfl, "m": w.m, "levels": w.levels, "relax": w.relax,
                   "psi_widths": list(w.psi_widths), "tol": w.tol, "iterations": K,
                   "cycle": args.cycle, "boundary": getattr(w, "boundary", "periodic"),
                   "time_to_residual_ms": round(ms, 4),
                   "final_residual": res["history"][-1],
                   "history": [float(f"{h:.4e}") for h in res["history"]],
                   "final_sweep": args.final_sweep,
                   "parallelism": f"replicas{world}",
                   "l2": "inputs larger than L2 (8 GiB state vs 126 MB L2)"},
        "roofline": {"bound": "alu", "kernel": s.describe() + " (fine FCF sweep)",
                     "achieved": round(achieved, 3), "peak": round(FP64_PEAK_TFLOPS, 2),
                     "unit": "TFLOP/s", "frac": round(achieved / FP64_PEAK_TFLOPS, 4),
                     "peak_note": "FP64 pipe: 64 DFMA/clk/SM x 148 x 1.965 GHz (derived from the "
                                  "guide's unit count and the max clock; MEASURED_PEAKS.json has "
                                  "no FP64 entry)",
                     "probe": {"tflops": probe_tf, "sm_mhz": probe_mhz,
                               "frac": round(achieved / probe_tf, 4) if probe_tf else None,
                               "source": "profiles/r02_fp64_probe.json (tools/probe_fp64.sh)"},
                     "executed": executed,
                     "flops_note": f"{FLOPS_PER_POINT_STEP[w.tableau]:g} algorithmic flops per "
                                   "point-step (stage form, SURVEY 8d); the kernel issues fewer "
                                   "FP64 instructions (folded last stage, Shu-Osher SSP-RK3: "
                                   "DESIGN.md 6.1)",
                     # ncu DRAM bytes per launch of this kernel, captured on cfg5 only
                     "traffic": _profile_traffic() if w.name == "cfg5" else None,
                     "avg_launch_ms": round(avg_ms, 4), "launches": n_f,
                     "timed_pass": "a second timed region of the same K solves with per-launch "
                                   "CUDA events on the solver's stream ("
                                   f"{ms_total_prof / args.steps:.3f} ms/solve instrumented)",
                     "flops_per_launch": flops},
        "kernel_time_share": shares,
        "relax_kernel_rate": round(dof * world / (ms_f / max(args.steps, 1) / 1e3), 1) if ms_f else None,
        "coarse_solve": coarse,
        "gpu_launches": int(launches),
        "e2e": e2e,
    }
    if rank == 0:
        line["clocks"] = _clock_summary(clk_path, local)
        if not args.no_cpu_baseline and world == 1 and getattr(w, "boundary", "periodic") == "periodic":
            line["cpu_baseline"] = oracle_sample(w, args.cpu_budget)
            line["cpu_sequential"] = sequential_sample(w, args.cpu_budget / 2)
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_shard(args, w):
    """--mode shard: one problem split into N contiguous time blocks, one per GPU
    (mgrit_solve_shard); value = the problem's fine DOF updates / the
    max-over-ranks device time (strong scaling)."""
    import torch
    from paper_1910_03726_b200 import build as B
    from paper_1910_03726_b200 import problem, timeshard

    dist, rank, world = _dist()
    B.build()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    psi = problem.psi_inputs(w)
    sh = timeshard.ShardSolver(w, psi, rank, world, stream=stream)
    comm = timeshard.TorchDistComm(sh.send_stage, sh.recv_stage, stream) if world > 1 else None
    guess = sh.local_guess()
    out = torch.empty_like(guess)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        res = sh.solve(comm, guess, w.tol, w.max_iter, out=out)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        res = sh.solve(comm, guess, w.tol, w.max_iter, out=out)
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_local = e0.elapsed_time(e1) / args.steps
    K = res["iterations"]
    dof = problem.dof_updates(w, K)
    ms = ms_local
    if dist:
        t = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        line = {"metric": METRIC, "value": dof / (ms / 1e3), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "mode": "shard",
                "config": {"workload": w.name, "nx": w.nx, "nt": w.nt, "m": w.m,
                           "levels": w.levels, "relax": w.relax, "iterations": K,
                           "history": [float(f"{h:.4e}") for h in res["history"]],
                           "parallelism": f"time{world}",
                           "l2": "inputs larger than L2"},
                "e2e": None}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args, w):
    dist, rank, world = _dist()
    if rank != 0:
        return
    vals = []
    samp = None
    for it in range(args.warmup + args.steps):
        samp = oracle_sample(w, args.cpu_budget / 2)
        if it >= args.warmup:
            vals.append(samp["value"])
    v = sum(vals) / len(vals)
    samp["value"] = v
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": w.name, "nx": w.nx, "nt": w.nt, "scheme": f"{w.tableau}+U{w.order}",
                       "m": w.m, "levels": w.levels, "relax": w.relax},
            "cpu_baseline": samp,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5", choices=sorted(W.ALL))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-prof", action="store_true",
                    help="time without the per-launch CUDA events (no roofline / shares)")
    ap.add_argument("--final-sweep", default="predict", choices=["off", "predict", "always"],
                    help="mgrit_set_final_sweep mode (include/mgrit.h)")
    ap.add_argument("--cycle", default="V", choices=["V", "F"],
                    help="multilevel cycle (DESIGN.md R19); the bench line is the V-cycle")
    ap.add_argument("--mode", default="replicas", choices=["replicas", "shard"],
                    help="N > 1: independent replicas (default, weak scaling) or one problem "
                         "in N time blocks (mgrit_solve_shard, strong scaling; DESIGN.md §7)")
    ap.add_argument("--opt", action="append", default=[], metavar="NAME=V1,V2",
                    help="mgrit_set_option override (experiments), e.g. fine_tile=128,15")
    args = ap.parse_args()
    w = W.ALL[args.config]
    if args.impl == "reference":
        run_reference(args, w)
    elif args.mode == "shard":
        run_shard(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()

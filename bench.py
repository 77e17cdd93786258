#!/usr/bin/env python
"""Benchmark of the pffmg hot path (BASELINE.json metric) -- one JSON line.

Headline workload: cfg2 (BASELINE configs[1]) -- 2D notched square, 1024^2 Q1
quads, 3,151,875 fp64 DoFs, NoSplit, 8-level GMG, Chebyshev degree 3.

* a "step" is one application of the linearised monolithic Jacobian (vmult,
  the north-star kernel) to a seeded N(0,1) vector, inputs resident in HBM,
  L2 flushed (512 MiB write) before every step; timed with CUDA events on the
  launching stream.  value = GDoF/s = DoFs x steps / sum(step time), summed
  over ranks (max-over-ranks time).
* e2e: the same metric through the public API `PhaseFieldOperator.apply`
  with pinned host buffers (H2D of v, kernel, D2H of the result inside the
  timed region).
* solve: one Newton-step linear solve (build_level_contexts + GMRES(30) to
  rel 1e-8 with the V(1,1) GMG preconditioner), the second half of the metric.
* roofline: achieved = B_C (SURVEY §8d algorithmic bytes of the reference's
  cached-coefficient vmult) / kernel time; B_F (the recompute model this
  kernel implements) and ncu DRAM bytes reported beside it.
* cpu_baseline: the CPU oracle port of the reference vmult on the host cores.

`--impl reference` times the CPU oracle port (the reference is pure Python
and cannot travel to the box) on the same workload and prints the same line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PFF Jacobian vmult GDoF/s and GMG-GMRES solve time/Newton step, % HBM roofline"
FP64_PEAK_TFLOPS = 34.2     # B200 FP64 FMA throughput measured with tools/microbench.cu


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def algorithmic_bytes(dim, V, C, Q=None):
    """B_C (cached tables, the reference algorithm) and B_F (recompute);
    Q = quadrature points per cell (2^dim for Q1, 9 for the Q2 cfg3)."""
    nc, Q = dim + 1, (Q or 2 ** dim)
    b_c = 16 * nc * V + 8 * Q * (2 + dim * (dim + 1) // 2) * C + nc * V
    b_f = 8 * (3 * nc + 1) * V + nc * V
    return b_c, b_f


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except (ValueError, IndexError):
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_vmult_rate(prob, threads, reps):
    """Oracle port of the reference vmult (oracle/, CPU): GDoF/s, median of reps."""
    from oracle import fe, jacobian, meshgen
    levels = meshgen.build_hierarchy(prob.blocks, prob.n_levels, prob.dim)
    T = fe.LevelTables(levels[-1], prob.n_levels - 1)
    p = prob.params
    mat = jacobian.Material(mu=p.mu, lam=p.lam, g_c=p.g_c, kappa=p.kappa, eps=p.eps)
    st = jacobian.State(U=prob.state.U, U_prev1=prob.state.U, U_prev2=prob.state.U, t=0.0,
                        t_prev1=0.0, t_prev2=0.0, phi_tilde=prob.state.phi_tilde)
    mask = prob.dirichlet.is_constrained | prob.active
    t0 = time.perf_counter()
    op = jacobian.JacobianOperator(T, st, mask, mat, threads=threads)
    t_cache = time.perf_counter() - t0
    op.apply(prob.v)                                      # warm
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        op.apply(prob.v)
        ts.append(time.perf_counter() - t0)
    return prob.n_dofs / float(np.median(ts)) * 1e-9, float(np.median(ts)), t_cache, ts


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1902_08112_b200 import configs
    prob = configs.make(args.config)
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    rate, med, t_cache, ts = cpu_vmult_rate(prob, threads, args.warmup + args.steps)
    steps = ts[args.warmup:]
    per = float(np.mean(steps))
    value = prob.n_dofs / per * 1e-9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GDoF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY §8d)",
        "config": {"workload": (f"{args.config} vmult" if args.gpus <= 1 else
                                f"{args.config} x{args.gpus} stacked vmult (CPU sample: one {args.config} "
                                f"square; the CPU rate per DoF does not depend on the stacking)"),
                   "n_dofs": prob.n_dofs},
        "cpu_baseline": {"value": value, "unit": "GDoF/s", "cores": threads, "kind": "port",
                         "sample": f"{args.config} full-size vmult x{args.steps} (oracle/ numpy "
                                   f"restatement of model.py:368-375, {threads} threads); "
                                   f"coefficient cache build {t_cache:.2f}s excluded"},
        "e2e": {"value": value, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_gpu(args):
    import torch
    ws, rank, local = dist_env()
    local = local % max(torch.cuda.device_count(), 1)   # --backend gloo smoke runs share one GPU
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        # one collective over every rank before the first point-to-point halo
        # batch (batch_isend_irecv must not be a communicator's first operation)
        dist.all_reduce(torch.zeros(1, device="cuda") if args.backend == "nccl" else torch.zeros(1))
    from paper_1902_08112_b200 import _lib, configs, krylov, mgsolve
    from paper_1902_08112_b200.model import ConstraintMask, PhaseFieldOperator, SplitKind

    if ws > 1 and args.config == "cfg2":
        # weak scaling: one cfg2 slab (1024^2 cells) per GPU, stacked in y
        prob = configs.notched_square(8, 3, "cfg2", stack=ws)
    else:
        prob = configs.make(args.config)
    mesh = prob.disc.hierarchy.finest
    mask = prob.dirichlet.combined_with(prob.active, np.zeros(prob.n_dofs))
    cmask = ConstraintMask(mask.is_constrained, mask.inhomogeneity)
    n = prob.n_dofs
    if ws > 1:
        from paper_1902_08112_b200 import distributed as D
        from paper_1902_08112_b200.lattice import info_from_mesh
        levels = prob.disc.hierarchy.levels
        part = D.SlabPartition([int(info_from_mesh(m).ncell[-1]) for m in levels], ws, rank,
                               order=getattr(info_from_mesh(mesh), "order", 1))
        dop = D.DistributedOperator(mesh, len(levels) - 1, part, prob.state, cmask, prob.params,
                                    SplitKind.NOSPLIT)
        op = dop.local
        v = torch.as_tensor(dop.to_local(prob.v), device="cuda")
        out = torch.empty_like(v)

        def step():                       # halo exchange (NCCL) + fused vmult of the owned rows
            dop.apply_local(v, out)
    else:
        op = PhaseFieldOperator(prob.disc.finest, prob.state, cmask, prob.params, SplitKind.NOSPLIT)
        v = torch.as_tensor(prob.v, device="cuda")
        out = torch.empty_like(v)

        def step():
            op.apply_dev(_lib.FULL, v, out)
    flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    def load_for(seconds):
        """Keep the GPU busy with the same work so nvidia-smi sees it under load."""
        t_end = time.perf_counter() + seconds
        while time.perf_counter() < t_end:
            for _ in range(20):
                flush.zero_()
                step()
            torch.cuda.synchronize()

    with Clocks(local) as clk:
        load_for(0.4)
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for e0, e1 in evs:
            flush.zero_()
            e0.record(stream)
            step()
            e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if ws > 1:
            torch.distributed.barrier()
        load_for(0.4)
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    t_tot = float(np.sum(step_ms)) * 1e-3
    if ws > 1:
        tt = torch.tensor([t_tot], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_tot = float(tt.item())
    per = t_tot / args.steps
    value = n / per * 1e-9                  # global DoFs per step (all ranks) / max-over-ranks time

    # ---------------------------------------------------------------- e2e
    if ws > 1:
        h_in = torch.from_numpy(dop.to_local(prob.v)).pin_memory()
        h_out = torch.empty(v.numel(), dtype=torch.float64).pin_memory()

        def e2e_call():
            v.copy_(h_in, non_blocking=True)
            step()
            h_out.copy_(out, non_blocking=True)
            torch.cuda.current_stream().synchronize()
    else:
        h_in = torch.from_numpy(prob.v.copy()).pin_memory()
        h_out = torch.empty(n, dtype=torch.float64).pin_memory()

        def e2e_call():
            op.apply(h_in, out=h_out)
            torch.cuda.synchronize()
    for _ in range(2):
        e2e_call()
    e2e_t = []
    for _ in range(max(3, min(args.steps, 20))):
        if ws > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        e2e_call()
        e2e_t.append(time.perf_counter() - t0)
    e2e_per = float(np.median(e2e_t))
    if ws > 1:
        tt = torch.tensor([e2e_per], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_per = float(tt.item())
    e2e_bytes = 8 * h_in.numel()

    # -------------------------------------------------------------- solve
    solve = None
    if not args.no_solve and ws == 1:
        from paper_1902_08112_b200 import model as M
        ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)
        cmask_dev = torch.as_tensor(mask.is_constrained, device="cuda")
        state_dev = M.LinearizationState(
            U=torch.as_tensor(prob.state.U, device="cuda"), U_prev1=torch.as_tensor(prob.state.U_prev1, device="cuda"),
            U_prev2=torch.as_tensor(prob.state.U_prev2, device="cuda"), t=prob.state.t,
            t_prev1=prob.state.t_prev1, t_prev2=prob.state.t_prev2,
            phi_tilde=torch.as_tensor(prob.state.phi_tilde, device="cuda"))
        # the Newton loop holds its Dirichlet data and active set on the device, like the state
        dirichlet_dev = M.ConstraintMask(torch.as_tensor(prob.dirichlet.is_constrained, device="cuda"),
                                         torch.as_tensor(prob.dirichlet.inhomogeneity, device="cuda"))
        active_dev = torch.as_tensor(prob.active, device="cuda")

        def newton_step():
            """One linear Newton step of ActiveSetSolver.solve_step (nonlinear.py:146-181):
            R~ = -A(U) with constrained rows zeroed, GMG setup, GMRES(30)."""
            t0 = time.perf_counter()
            R = M.residual(prob.disc.finest, state_dev, dirichlet_dev, prob.params, SplitKind.NOSPLIT)
            R.neg_()
            R[cmask_dev] = 0.0
            ctxs = mgsolve.build_level_contexts(prob.disc, state_dev, active_dev, dirichlet_dev,
                                                prob.params, SplitKind.NOSPLIT)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            pc = mgsolve.VCyclePreconditioner(ctxs, degree=prob.degree)
            x, its = krylov.gmres(ctxs[-1].op.apply, pc, R, ctl)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            return t1 - t0, t2 - t1, its

        newton_step()                                   # warm (graph capture, probes)
        runs = [newton_step() for _ in range(3)]
        setup_s = float(np.median([r[0] for r in runs]))
        gmres_s = float(np.median([r[1] for r in runs]))
        its = runs[-1][2]
        solve = {"setup_ms": setup_s * 1e3, "gmres_ms": gmres_s * 1e3, "gmres_iters": its,
                 "ms_per_newton_step": (setup_s + gmres_s) * 1e3,
                 "rhs": "Newton RHS -A(U), constrained rows zeroed, from the GPU residual kernel",
                 "resident": "state U, Dirichlet mask and active set on the device (as the Newton loop holds them)",
                 "control": "GMRES(30) rel 1e-8 abs 0, V(1,1) FULL, Chebyshev deg %d" % prob.degree,
                 "timing": "wall clock, median of 3 after one warm-up"}
    elif not args.no_solve and ws > 1:
        from paper_1902_08112_b200 import model as M
        from paper_1902_08112_b200.dist_solver import DistGMG
        ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)

        def newton_step():
            torch.distributed.barrier()
            t0 = time.perf_counter()
            gmg = DistGMG(prob.disc.hierarchy.levels, ws, rank, degree=prob.degree)
            gmg.setup(prob.state, prob.active, prob.dirichlet, prob.params, SplitKind.NOSPLIT)
            # Newton RHS -A(U) on the rank's slab (the state carries its ghost planes),
            # rows constrained by Dirichlet | active zeroed (nonlinear.py:146-160)
            b = torch.zeros(gmg.L[-1].n, dtype=torch.float64, device="cuda")
            gmg.ops[-1].semilinear_dev(b)
            b.neg_()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            x, its = gmg.gmres(b, ctl)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            tt = torch.tensor([t1 - t0, t2 - t1], device="cuda", dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            return float(tt[0]), float(tt[1]), its

        newton_step()
        setup_s, gmres_s, its = newton_step()
        solve = {"setup_ms": setup_s * 1e3, "gmres_ms": gmres_s * 1e3, "gmres_iters": its,
                 "ms_per_newton_step": (setup_s + gmres_s) * 1e3,
                 "rhs": "Newton RHS -A(U) from the GPU residual kernel on each slab, constrained rows zeroed",
                 "control": "slab-distributed GMRES(30) rel 1e-8 abs 0, V(1,1) FULL, Chebyshev deg %d, "
                            "%s halos + all-reduced dots" % (prob.degree, args.backend),
                 "timing": "wall clock, max over ranks"}

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return 0

    hbm, peak_kind = peaks()
    b_c, b_f = algorithmic_bytes(prob.dim, mesh.n_vertices, mesh.n_cells,
                                 9 if getattr(mesh, "order", 1) == 2 else None)
    traffic = flops = None
    prof = os.path.join(ROOT, "profiles", "ncu_vmult_cfg2_r1.json")   # this round's capture
    if os.path.exists(prof) and args.config == "cfg2":
        try:
            with open(prof) as f:
                pj = json.load(f)
            traffic = pj.get("dram_bytes_per_launch")
            flops = pj.get("fp64_flops_per_launch")
        except Exception:
            traffic = flops = None
    achieved = b_c / per * 1e-9
    peak_all = hbm * ws                           # aggregate over the ranks
    workload = (f"{args.config}: 2D notched square 1024^2 Q1 NoSplit vmult" if ws == 1 else
                f"{args.config} x{ws}: {ws} stacked 1024^2 notched squares (1024 x {1024 * ws} Q1), "
                f"y-slab per GPU, {args.backend} halo exchange + fused vmult") if args.config == "cfg2" else \
        {"cfg1": "cfg1: 2D notched square 64^2 Q1 NoSplit vmult",
         "cfg3": "cfg3: 2D pressurised cracks 512^2 Q2 (3x3 Gauss) NoSplit vmult, p = 1e-3",
         "cfg4": "cfg4: 3D L-prism 786k Q1 hexes NoSplit vmult",
         "cfg5": "cfg5: 3D cube 384^3 Q1 hexes NoSplit vmult"}.get(args.config, args.config)
    if ws > 1 and args.config != "cfg2":
        workload += f", strong scaling: {ws} slabs of the last axis, {args.backend} halo exchange"
    line = {
        "metric": METRIC, "value": value, "unit": "GDoF/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak" if (ws == 1 or args.config == "cfg2") else "strong", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded state/vector, SURVEY §8d; random-init, no dataset)",
        "config": {"workload": workload,
                   "n_dofs": n, "n_vertices": mesh.n_vertices, "n_cells": mesh.n_cells,
                   "l2": "flushed (512 MiB write) before every step",
                   "parallelism": f"slabs x{ws} (halo exchange)" if ws > 1 else "single GPU"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak_all, "unit": "GB/s",
                     "frac": achieved / peak_all, "traffic": traffic if ws == 1 else None,
                     "bytes_model": "B_C = 16 n_c V + 8 Q (2 + d(d+1)/2) C + n_c V (SURVEY §8d)",
                     "algorithmic_bytes_BC": b_c, "algorithmic_bytes_BF": b_f,
                     "frac_BF": b_f / per * 1e-9 / peak_all,
                     "frac_ncu": (traffic / per * 1e-9 / hbm) if (traffic and ws == 1) else None,
                     "peak_kind": peak_kind + (f" x{ws} GPUs" if ws > 1 else ""),
                     # the kernel recomputes the coefficient tables: its own ceiling is FP64
                     # issue; flops = SASS DFMA x2 + DADD + DMUL of the ncu capture
                     "fp64": ({"achieved": flops / per * 1e-12, "peak": FP64_PEAK_TFLOPS * ws,
                               "unit": "TFLOP/s", "frac": flops / per * 1e-12 / FP64_PEAK_TFLOPS,
                               "flops_per_launch": flops,
                               "peak_kind": "measured, tools/microbench.cu DFMA chains"}
                              if (flops and ws == 1) else None)},
        "e2e": {"value": n / e2e_per * 1e-9, "unit": "GDoF/s", "h2d_bytes_per_step": e2e_bytes,
                "d2h_bytes_per_step": e2e_bytes,
                "path": ("PhaseFieldOperator.apply(pinned host tensor, out=pinned host tensor)" if ws == 1
                         else "per rank: pinned H2D of the slab, halo exchange + vmult, D2H; bytes per rank")},
        # our kernels per step: the fused vmult; on a slab (N > 1) the interior rows
        # and, after the halo lands, the two boundary rows
        "gpu_launches": args.steps * (1 if ws == 1 else (3 if getattr(mesh, "order", 1) == 2 else 2)),
        "solve": solve,
        "wall_s_timed_region": wall,
        "step_ms_min_max": [float(np.min(step_ms)), float(np.max(step_ms))],
    }
    line["clocks"] = clk.summary()
    if not args.no_cpu and ws == 1:
        threads = os.cpu_count() or 1
        rate, med, t_cache, _ = cpu_vmult_rate(prob, threads, 3)
        line["cpu_baseline"] = {"value": rate, "unit": "GDoF/s", "cores": threads, "kind": "port",
                                "sample": f"{args.config} full-size vmult, median of 3 (oracle/ "
                                          f"numpy port of model.py:368-375, {threads} threads, "
                                          f"{med * 1e3:.0f} ms each)"}
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="pffmg", choices=["pffmg", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: host-staged communication, for functional runs of N>1 on one GPU")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())

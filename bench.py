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
* solve.hbm: sum of the algorithmic bytes of every kernel of one Newton step
  (tools/bytemodel.py over the eager launch list) / T_solve / P.
* configs: the same vmult + Newton step on cfg3 (Q2), cfg4 (3D L-prism) and
  cfg5 (3D cube 384^3, 228M DoFs, on one GPU).
* N > 1: `value` weak-scales the headline (one 1024^2 cfg2 slab per GPU, so
  the driver's per-N ratios are a like-for-like efficiency); the north
  star's strong scaling of the largest config is the `strong_scaling`
  sub-result -- cfg5 cut into N z-slabs (sharded vmult and a DistGMG
  Newton step), to be divided by configs.cfg5 of the N = 1 line.
* parity: the GPU vmult against the CPU arm's output of the same vector, and
  the Newton step's GMRES iterations / solution fingerprint against the
  reference's (tests/golden/configs_full.npz).
* cpu_baseline: the reference's CPU implementation on the host cores -- the
  unmodified fracmg from baseline/_ref (pip-installed in the build container,
  shipped with the snapshot) when present ("reference"), else the oracle/
  numpy port ("port", bit-equal to it).

`--impl reference` times that CPU arm on the same workload (vmult at all host
threads and at 1 thread, plus the Newton-step setup and GMRES wall clocks)
and prints the same line with the same config.
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


# ------------------------------------------------------------ CPU arm

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def import_reference():
    """The unmodified reference package (pip-installed into baseline/_ref in the
    build container; git-ignored, shipped with the snapshot), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "fracmg")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import fracmg  # noqa: F401
        from fracmg import fem, krylov, mesh, mgsolve, model  # noqa: F401
        return sys.modules["fracmg"]
    except Exception:
        return None


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


class CpuArm:
    """The reference's CPU implementation of the path on this host: the
    unmodified fracmg from baseline/_ref when it is installed (kind
    "reference"), else the oracle/ numpy port of it (kind "port"; bit-equal
    to the reference, tests/test_oracle_fullsize.py)."""

    def __init__(self, prob):
        self.prob = prob
        fr = import_reference()
        self.kind = "reference" if fr is not None else "port"
        p, s = prob.params, prob.state
        if fr is not None:
            from fracmg import fem, mesh
            from fracmg import model as rm
            hier = mesh._build_hierarchy(prob.blocks, prob.n_levels, prob.dim,
                                         lambda lo, hi, ax, sd: np.zeros(len(lo)))
            self.disc = fem.Discretization(hier)
            self.state = rm.LinearizationState(U=s.U, U_prev1=s.U_prev1, U_prev2=s.U_prev2, t=s.t,
                                               t_prev1=s.t_prev1, t_prev2=s.t_prev2, phi_tilde=s.phi_tilde)
            self.params = rm.MaterialParams(mu=p.mu, lam=p.lam, g_c=p.g_c, kappa=p.kappa, eps=p.eps)
            self.dirichlet = fem.ConstraintMask(prob.dirichlet.is_constrained, prob.dirichlet.inhomogeneity)
        else:
            from oracle import fe, jacobian, meshgen
            levels = meshgen.build_hierarchy(prob.blocks, prob.n_levels, prob.dim)
            self.levels = levels
            self.tables = [fe.LevelTables(m, l) for l, m in enumerate(levels)]
            self.transfers = fe.Transfers(levels)
            self.mat = jacobian.Material(mu=p.mu, lam=p.lam, g_c=p.g_c, kappa=p.kappa, eps=p.eps)
            self.st = jacobian.State(U=s.U, U_prev1=s.U_prev1, U_prev2=s.U_prev2, t=s.t,
                                     t_prev1=s.t_prev1, t_prev2=s.t_prev2, phi_tilde=s.phi_tilde)

    @property
    def what(self):
        return ("fracmg (the unmodified reference, baseline/_ref)" if self.kind == "reference"
                else "oracle/ numpy port of the reference")

    def operator(self, threads):
        prob = self.prob
        mask = prob.dirichlet.is_constrained | prob.active
        if self.kind == "reference":
            from fracmg import fem
            from fracmg import model as rm
            return rm.PhaseFieldOperator(self.disc.finest, self.state, fem.ConstraintMask(mask, np.zeros(mask.size)),
                                         self.params, rm.SplitKind.NOSPLIT, threads=threads)
        from oracle import jacobian
        return jacobian.JacobianOperator(self.tables[-1], self.st, mask, self.mat, threads=threads)

    def vmult(self, threads, reps):
        """Median-timed applies of the seeded vector (cache build excluded)."""
        t0 = time.perf_counter()
        op = self.operator(threads)
        t_cache = time.perf_counter() - t0
        out = op.apply(self.prob.v)                       # warm
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            op.apply(self.prob.v)
            ts.append(time.perf_counter() - t0)
        return out, ts, t_cache

    def newton_rhs(self, threads):
        prob = self.prob
        mask = prob.dirichlet.is_constrained | prob.active
        if self.kind == "reference":
            from fracmg import model as rm
            R = -rm.residual(self.disc.finest, self.state, self.dirichlet, self.params, rm.SplitKind.NOSPLIT,
                             threads=threads)
        else:
            from oracle import jacobian
            R = -jacobian.residual(self.tables[-1], self.st, prob.dirichlet.is_constrained, self.mat)
        R[mask] = 0.0
        return R

    def setup(self, threads):
        prob = self.prob
        if self.kind == "reference":
            from fracmg import mgsolve
            from fracmg import model as rm
            return mgsolve.build_level_contexts(self.disc, self.state, prob.active, self.dirichlet, self.params,
                                                rm.SplitKind.NOSPLIT, threads=threads)
        from oracle import solvers
        return solvers.build_levels(self.transfers, self.tables, self.st, prob.active,
                                    prob.dirichlet.is_constrained, self.mat, "none", threads=threads)

    def gmres(self, ctxs, R, max_iters=1000):
        deg = self.prob.degree
        if self.kind == "reference":
            from fracmg import krylov, mgsolve
            ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=max_iters)
            pc = lambda v: mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, v, degree=deg)  # noqa: E731
            try:
                return krylov.gmres(ctxs[-1].op.apply, pc, R, ctl)
            except krylov.NoConvergence as e:
                return e.x, e.iterations
        from oracle import solvers
        ctl = solvers.Control(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=max_iters)
        try:
            return solvers.gmres(ctxs[-1].op.apply, lambda v: solvers.vcycle(ctxs, v, "full", degree=deg), R, ctl)
        except solvers.NoConvergence as e:
            return e.x, e.iterations

    def solve(self, threads, full=True):
        """Wall clocks of build_level_contexts and gmres.  With
        full=False a bounded sample: setup plus ONE preconditioned GMRES
        iteration; the Newton step is extrapolated as setup + its x (one
        iteration minus the restart's true-residual vmult)."""
        R = self.newton_rhs(threads)
        t0 = time.perf_counter()
        ctxs = self.setup(threads)
        t_setup = time.perf_counter() - t0
        if full:
            t0 = time.perf_counter()
            x, its = self.gmres(ctxs, R)
            return {"threads": threads, "setup_s": t_setup, "gmres_s": time.perf_counter() - t0,
                    "gmres_iters": int(its), "newton_step_s": t_setup + time.perf_counter() - t0,
                    "sample": "full Newton-step solve"}
        t0 = time.perf_counter()
        self.gmres(ctxs, R, max_iters=1)
        t_one = time.perf_counter() - t0
        t0 = time.perf_counter()
        ctxs[-1].op.apply(R)
        t_v = time.perf_counter() - t0
        return {"threads": threads, "setup_s": t_setup, "gmres_iter_s": t_one - t_v,
                "sample": "setup + one GMRES(30) iteration (V-cycle + vmult + MGS); "
                          "gmres_s extrapolated = iterations x gmres_iter_s"}


def config_dict(args, ws, prob, mesh):
    """The workload description both arms print (same_config)."""
    name = args.config
    if name == "cfg2" and ws > 1:
        workload = (f"{name} x{ws}: {ws} stacked 1024^2 notched squares (1024 x {1024 * ws} Q1), "
                    f"y-slab per GPU, halo exchange + fused vmult")
    else:
        workload = {"cfg1": "cfg1: 2D notched square 64^2 Q1 NoSplit vmult",
                    "cfg2": "cfg2: 2D notched square 1024^2 Q1 NoSplit vmult",
                    "cfg3": "cfg3: 2D pressurised cracks 512^2 Q2 (3x3 Gauss) NoSplit vmult, p = 1e-3",
                    "cfg4": "cfg4: 3D L-prism 786k Q1 hexes NoSplit vmult",
                    "cfg5": "cfg5: 3D cube 384^3 Q1 hexes NoSplit vmult"}[name]
        if ws > 1:
            workload += f", strong scaling: {ws} slabs of the last axis, halo exchange"
    return {"workload": workload, "n_dofs": prob.n_dofs, "n_vertices": mesh.n_vertices,
            "n_cells": mesh.n_cells, "l2": "flushed (512 MiB write) before every GPU step",
            "parallelism": f"slabs x{ws} (halo exchange)" if ws > 1 else "single GPU"}


def problem_for(args, ws):
    from paper_1902_08112_b200 import configs
    if ws > 1 and args.config == "cfg2":
        # weak scaling: one cfg2 slab (1024^2 cells) per GPU, stacked in y
        return configs.notched_square(8, 3, "cfg2", stack=ws)
    return configs.make(args.config)


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    prob = problem_for(args, 1)
    mesh = prob.disc.hierarchy.finest
    arm = CpuArm(prob)
    threads = os.cpu_count() or 1
    _, ts, t_cache = arm.vmult(threads, args.warmup + args.steps)
    steps = ts[args.warmup:]
    per = float(np.mean(steps))
    value = prob.n_dofs / per * 1e-9
    _, ts1, t_cache1 = arm.vmult(1, 3)
    solve = None
    if not args.no_solve and args.config in ("cfg1", "cfg2"):
        solve = {"all_threads": arm.solve(threads, full=True), "one_thread": arm.solve(1, full=False)}
        o = solve["one_thread"]
        o["gmres_iters"] = solve["all_threads"]["gmres_iters"]
        o["gmres_s"] = o["gmres_iter_s"] * o["gmres_iters"]
        o["newton_step_s"] = o["setup_s"] + o["gmres_s"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GDoF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak" if (ws == 1 or args.config == "cfg2") else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY §8d)",
        "config": config_dict(args, ws, problem_for(args, ws) if ws > 1 else prob,
                              (problem_for(args, ws) if ws > 1 else prob).disc.hierarchy.finest),
        "cpu_baseline": {"value": value, "unit": "GDoF/s", "cores": threads, "kind": arm.kind,
                         "sample": f"{args.config} full-size vmult x{args.steps} ({arm.what}, "
                                   f"PhaseFieldOperator.apply, model.py:368-375, {threads} threads"
                                   + (f"; on N={ws} the per-DoF rate of one {args.config} square" if ws > 1 else "")
                                   + f"); coefficient cache build {t_cache:.2f}s excluded",
                         "cpu_model": cpu_model(),
                         "one_thread": {"value": prob.n_dofs / float(np.median(ts1)) * 1e-9,
                                        "ms": float(np.median(ts1)) * 1e3, "cache_build_s": t_cache1}},
        "solve": solve,
        "e2e": {"value": value, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def golden_full(tag):
    """Reference fingerprints of a full-size config (tests/golden/configs_full.npz,
    made by the reference itself), or None."""
    path = os.path.join(ROOT, "tests", "golden", "configs_full.npz")
    if not os.path.exists(path):
        return None
    z = np.load(path)
    return {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(tag + "/")} or None


def fingerprint_err(x, g, key):
    """Relative error of x's sampled entries vs the reference's (make_golden.sample_index)."""
    if g is None or f"{key}_sample" not in g:
        return None
    x = np.asarray(x, dtype=float)
    idx = np.sort(np.random.default_rng(11).choice(x.size, size=min(x.size, 4096), replace=False))
    ref = g[f"{key}_sample"]
    return float(np.linalg.norm(x[idx] - ref) / np.linalg.norm(ref))


def src_sha():
    """Hash of the CUDA sources + header + build flags: what a profile was captured from."""
    import hashlib
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_1902_08112_b200", "csrc")
    for f in sorted(os.listdir(csrc)):
        if f.endswith((".cu", ".cuh")) or f == "Makefile":
            with open(os.path.join(csrc, f), "rb") as fh:
                h.update(f.encode() + fh.read())
    with open(os.path.join(ROOT, "include", "pffmg.h"), "rb") as fh:
        h.update(fh.read())
    return h.hexdigest()[:16]


def profile_for(config):
    """ncu summary of this config's vmult kernel captured from the current sources
    (profiles/ncu_vmult_<cfg>_r*.json with a matching src_sha), newest round first."""
    import glob
    cur = src_sha()
    best = None
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", f"ncu_vmult_{config}_r*.json"))):
        try:
            with open(p) as f:
                pj = json.load(f)
        except Exception:
            continue
        best = (p, pj)
        if pj.get("src_sha") == cur:
            return os.path.basename(p), pj, True
    if best:
        return os.path.basename(best[0]), best[1], False
    return None, None, False


def time_steps(step, steps, warmup, flush, stream, sync=None):
    """CUDA-event times (ms) of `steps` flushed steps after `warmup` (>= 3) warm ones."""
    import torch
    for _ in range(max(warmup, 3)):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if sync:
        sync()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for e0, e1 in evs:
        flush.zero_()
        e0.record(stream)
        step()
        e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if sync:
        sync()
    return [e0.elapsed_time(e1) for e0, e1 in evs], wall


def newton_step_fn(prob, mask):
    """One linear Newton step of ActiveSetSolver.solve_step (nonlinear.py:146-181):
    R~ = -A(U) with constrained rows zeroed (GPU residual), GMG setup, GMRES(30)
    rel 1e-8, with the state / Dirichlet data / active set resident on the device."""
    import torch
    from paper_1902_08112_b200 import krylov, mgsolve
    from paper_1902_08112_b200 import model as M
    ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)
    cmask_dev = torch.as_tensor(mask.is_constrained, device="cuda")
    s = prob.state
    state_dev = M.LinearizationState(
        U=torch.as_tensor(s.U, device="cuda"), U_prev1=torch.as_tensor(s.U_prev1, device="cuda"),
        U_prev2=torch.as_tensor(s.U_prev2, device="cuda"), t=s.t, t_prev1=s.t_prev1, t_prev2=s.t_prev2,
        phi_tilde=torch.as_tensor(s.phi_tilde, device="cuda"))
    dirichlet_dev = M.ConstraintMask(torch.as_tensor(prob.dirichlet.is_constrained, device="cuda"),
                                     torch.as_tensor(prob.dirichlet.inhomogeneity, device="cuda"))
    active_dev = torch.as_tensor(prob.active, device="cuda")

    def newton_step():
        t0 = time.perf_counter()
        R = M.residual(prob.disc.finest, state_dev, dirichlet_dev, prob.params, M.SplitKind.NOSPLIT)
        R.neg_()
        R[cmask_dev] = 0.0
        ctxs = mgsolve.build_level_contexts(prob.disc, state_dev, active_dev, dirichlet_dev,
                                            prob.params, M.SplitKind.NOSPLIT)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        pc = mgsolve.VCyclePreconditioner(ctxs, degree=prob.degree)
        x, its = krylov.gmres(ctxs[-1].op.apply, pc, R, ctl)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1, its, x

    return newton_step


def newton_step_numpy_fn(prob, mask):
    """The same Newton step with numpy state, masks and right-hand side in and a
    numpy solution out -- what the reference's own driver (ActiveSetSolver.solve_step
    through patch.install) exchanges with the twins every step."""
    from paper_1902_08112_b200 import krylov, mgsolve
    from paper_1902_08112_b200 import model as M
    ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)

    def newton_step():
        t0 = time.perf_counter()
        R = M.residual(prob.disc.finest, prob.state, prob.dirichlet, prob.params, M.SplitKind.NOSPLIT)
        R = -np.asarray(R)
        R[mask.is_constrained] = 0.0
        ctxs = mgsolve.build_level_contexts(prob.disc, prob.state, prob.active, prob.dirichlet,
                                            prob.params, M.SplitKind.NOSPLIT)
        pc = mgsolve.VCyclePreconditioner(ctxs, degree=prob.degree)
        x, its = krylov.gmres(ctxs[-1].op.apply, pc, R, ctl)
        assert isinstance(x, np.ndarray)
        return time.perf_counter() - t0, its

    return newton_step


def solve_bytes(newton_step):
    """Algorithmic bytes and launches of one Newton step, from the launch list of
    an eager run (PFFMG_GRAPHS=0: the kernels the graphs replay) through
    tools/bytemodel.Recorder."""
    from paper_1902_08112_b200 import mgsolve
    from tools.bytemodel import Recorder
    old = os.environ.get("PFFMG_GRAPHS")
    os.environ["PFFMG_GRAPHS"] = "0"
    mgsolve._Session._cache.clear()
    mgsolve._NativeCycle._cache.clear()
    try:
        with Recorder() as rec:
            newton_step()
    finally:
        if old is None:
            os.environ.pop("PFFMG_GRAPHS", None)
        else:
            os.environ["PFFMG_GRAPHS"] = old
        mgsolve._Session._cache.clear()
        mgsolve._NativeCycle._cache.clear()
    return rec.summary()


def measure_solve(prob, mask, hbm, with_bytes=True):
    import torch
    newton_step = newton_step_fn(prob, mask)
    newton_step()                                   # warm (graph capture, probes)
    runs = [newton_step() for _ in range(5 if with_bytes else 3)]
    setup_s = float(np.median([r[0] for r in runs]))
    gmres_s = float(np.median([r[1] for r in runs]))
    its = runs[-1][2]
    x = runs[-1][3]
    out = {"setup_ms": setup_s * 1e3, "gmres_ms": gmres_s * 1e3, "gmres_iters": its,
           "ms_per_newton_step": (setup_s + gmres_s) * 1e3,
           "rhs": "Newton RHS -A(U), constrained rows zeroed, from the GPU residual kernel",
           "resident": "state U, Dirichlet mask and active set on the device (as the Newton loop holds them)",
           "control": "GMRES(30) rel 1e-8 abs 0, V(1,1) FULL, Chebyshev deg %d" % prob.degree,
           "timing": "wall clock, median of %d after one warm-up" % len(runs),
           "ms_per_newton_step_runs": [round((r[0] + r[1]) * 1e3, 3) for r in runs]}
    if with_bytes:
        step_np = newton_step_numpy_fn(prob, mask)
        step_np()
        ts = [step_np() for _ in range(3)]
        out["numpy_io"] = {"ms_per_newton_step": float(np.median([t[0] for t in ts])) * 1e3,
                           "gmres_iters": ts[-1][1],
                           "what": "the same step with numpy state / masks / right-hand side in and a numpy "
                                   "solution out (the reference driver's calling convention; pageable copies "
                                   "through pffmg_copy_h2d / _d2h)"}
        b = solve_bytes(newton_step)
        t = setup_s + gmres_s
        out["hbm"] = {"bytes_F": b["bytes_F"], "bytes_C": b["bytes_C"], "launches": b["launches"],
                      "frac_F": b["bytes_F"] / t * 1e-9 / hbm, "frac_C": b["bytes_C"] / t * 1e-9 / hbm,
                      "unmodelled": b["unmodelled"],
                      "top": {k: v for k, v in list(b["by_name"].items())[:6]},
                      "model": "tools/bytemodel.py: per launch, every vector read/written once + flags + "
                               "the state the kernels recompute from (F) or the reference's cached tables (C); "
                               "sum over the eager launch list of one Newton step / T_solve / P"}
    torch.cuda.synchronize()
    return out, x


def measure_config(name, hbm, steps=20, solve=True):
    """vmult + Newton step of another BASELINE config (sub-result of the bench line)."""
    import torch
    from paper_1902_08112_b200 import _lib, configs
    from paper_1902_08112_b200.model import ConstraintMask, PhaseFieldOperator, SplitKind
    prob = configs.make(name)
    mesh = prob.disc.hierarchy.finest
    mask = prob.dirichlet.combined_with(prob.active, np.zeros(prob.n_dofs))
    op = PhaseFieldOperator(prob.disc.finest, prob.state, ConstraintMask(mask.is_constrained, mask.inhomogeneity),
                            prob.params, SplitKind.NOSPLIT)
    v = torch.as_tensor(prob.v, device="cuda")
    out = torch.empty_like(v)
    flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
    ms, _ = time_steps(lambda: op.apply_dev(_lib.FULL, v, out), steps, 3, flush, torch.cuda.current_stream())
    per = float(np.mean(ms)) * 1e-3
    b_c, b_f = algorithmic_bytes(prob.dim, mesh.n_vertices, mesh.n_cells,
                                 9 if getattr(mesh, "order", 1) == 2 else None)
    del v, out
    solve, x = measure_solve(prob, mask, hbm, with_bytes=False) if solve else (None, None)
    g = golden_full(name)
    res = {"vmult_ms": per * 1e3, "value": prob.n_dofs / per * 1e-9, "unit": "GDoF/s",
           "frac_BC": b_c / per * 1e-9 / hbm, "frac_BF": b_f / per * 1e-9 / hbm, "n_dofs": prob.n_dofs}
    # this config's ncu capture (profiles/ncu_vmult_<cfg>_r*.json) when it was
    # taken from the current sources: DRAM traffic and FP64 rate of the kernel
    prof_name, pj, fresh = profile_for(name)
    if pj and fresh:
        traffic, flops = pj.get("dram_bytes_per_launch"), pj.get("fp64_flops_per_launch")
        res["profile"] = {"file": prof_name, "traffic": traffic,
                          "frac_ncu": traffic / per * 1e-9 / hbm if traffic else None,
                          "fp64_tflops": flops / per * 1e-12 if flops else None,
                          "fp64_frac": flops / per * 1e-12 / FP64_PEAK_TFLOPS if flops else None,
                          "kernel_us_ncu": (pj.get("kernels") or [{}])[0].get("duration_us")}
    if solve is not None:
        res.update({"newton_step_ms": solve["ms_per_newton_step"], "setup_ms": solve["setup_ms"],
                    "gmres_ms": solve["gmres_ms"], "gmres_iters": solve["gmres_iters"],
                    "gmres_iters_ref": int(g["gmres_iters"]) if g is not None else None,
                    "gmres_x_fingerprint_err": fingerprint_err(x.cpu().numpy(), g, "gmres_x")})
    if name == "cfg3":
        res["parity_note"] = "Q2: no reference implementation (parity unpinned; oracle/q2.py known-answer pins)"
    if name == "cfg5":
        res["note"] = ("384^3: the reference fingerprint exists at 96^3 and 192^3 (tests/test_gpu_fullsize.py); "
                       "the single-GPU figure the strong-scaling runs divide by")
    del op, flush, x
    from paper_1902_08112_b200 import mgsolve
    mgsolve._Session._cache.clear()
    mgsolve._NativeCycle._cache.clear()
    torch.cuda.empty_cache()
    torch.cuda.empty_cache()
    return res


def measure_strong(name, ws, rank, args):
    """Strong scaling of the north-star's largest configuration:
    cfg5 (384^3, 228M DoFs) cut into ws z-slabs, one per GPU -- the sharded
    fused vmult (halo exchange overlapped with the interior planes) and one
    slab-distributed Newton-step solve (DistGMG).  Times are max over ranks;
    the single-GPU reference is configs.cfg5 of the N = 1 line."""
    import torch
    from paper_1902_08112_b200 import configs, krylov
    from paper_1902_08112_b200 import distributed as D
    from paper_1902_08112_b200.lattice import info_from_mesh
    from paper_1902_08112_b200.model import ConstraintMask, SplitKind
    prob = configs.make(name)
    mesh = prob.disc.hierarchy.finest
    levels = prob.disc.hierarchy.levels
    mask = prob.dirichlet.combined_with(prob.active, np.zeros(prob.n_dofs))
    part = D.SlabPartition([int(info_from_mesh(m).ncell[-1]) for m in levels], ws, rank)
    dop = D.DistributedOperator(mesh, len(levels) - 1, part, prob.state,
                                ConstraintMask(mask.is_constrained, mask.inhomogeneity), prob.params,
                                SplitKind.NOSPLIT)
    v = torch.as_tensor(dop.to_local(prob.v), device="cuda")
    out = torch.empty_like(v)
    flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
    ms, _ = time_steps(lambda: dop.apply_local(v, out), args.steps, args.warmup, flush,
                       torch.cuda.current_stream(), lambda: torch.distributed.barrier())
    tt = torch.tensor([float(np.mean(ms))], device="cuda", dtype=torch.float64)
    torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
    per = float(tt.item()) * 1e-3
    res = {"config": name, "n_dofs": prob.n_dofs, "n_gpus": ws, "vmult_ms": per * 1e3,
           "value": prob.n_dofs / per * 1e-9, "unit": "GDoF/s",
           "what": "z-slab sharded fused vmult, halo exchange overlapped with the interior planes, "
                   f"time = max over ranks (the single-GPU figure: configs.{name} of the N = 1 line)"}
    del v, out, dop, flush
    torch.cuda.empty_cache()
    if not args.no_solve:
        from paper_1902_08112_b200.dist_solver import DistGMG
        ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)

        def newton_step():
            torch.distributed.barrier()
            t0 = time.perf_counter()
            gmg = DistGMG(levels, ws, rank, degree=prob.degree)
            gmg.setup(prob.state, prob.active, prob.dirichlet, prob.params, SplitKind.NOSPLIT)
            b = torch.zeros(gmg.L[-1].n, dtype=torch.float64, device="cuda")
            gmg.ops[-1].semilinear_dev(b)
            b.neg_()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            x, its = gmg.gmres(b, ctl)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            t = torch.tensor([t1 - t0, t2 - t1], device="cuda", dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            del gmg, x, b
            return float(t[0]), float(t[1]), its

        newton_step()
        setup_s, gmres_s, its = newton_step()
        res["newton_step"] = {"setup_ms": setup_s * 1e3, "gmres_ms": gmres_s * 1e3, "gmres_iters": its,
                              "ms": (setup_s + gmres_s) * 1e3,
                              "control": "slab-distributed GMRES(30) rel 1e-8, V(1,1) FULL, CGS2 Arnoldi, "
                                         "wall clock max over ranks"}
    return res


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
    from paper_1902_08112_b200 import _lib, krylov
    from paper_1902_08112_b200.model import ConstraintMask, PhaseFieldOperator, SplitKind

    prob = problem_for(args, ws)
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

        def step():                       # halo exchange + fused vmult of the owned rows
            dop.apply_local(v, out)
    else:
        op = PhaseFieldOperator(prob.disc.finest, prob.state, cmask, prob.params, SplitKind.NOSPLIT)
        v = torch.as_tensor(prob.v, device="cuda")
        out = torch.empty_like(v)

        def step():
            op.apply_dev(_lib.FULL, v, out)
    flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    def load_for(seconds):
        """Keep the GPU busy with the same work so nvidia-smi sees it under load.
        With several ranks every step is a halo exchange, so all ranks must run
        the same number of steps: they agree after every batch (max over ranks
        of "my time is not up yet") instead of each watching its own clock."""
        t_end = time.perf_counter() + seconds
        more = True
        while more:
            for _ in range(20):
                flush.zero_()
                step()
            torch.cuda.synchronize()
            more = time.perf_counter() < t_end
            if ws > 1:
                f = torch.tensor([1.0 if more else 0.0], device="cuda" if args.backend == "nccl" else "cpu")
                torch.distributed.all_reduce(f, op=torch.distributed.ReduceOp.MAX)
                more = bool(f.item() > 0.0)

    barrier = (lambda: torch.distributed.barrier()) if ws > 1 else None
    with Clocks(local) as clk:
        load_for(0.4)
        step_ms, wall = time_steps(step, args.steps, args.warmup, flush, stream, barrier)
        load_for(0.4)
    t_tot = float(np.sum(step_ms)) * 1e-3
    if ws > 1:
        tt = torch.tensor([t_tot], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_tot = float(tt.item())
    per = t_tot / args.steps
    value = n / per * 1e-9                  # global DoFs per step (all ranks) / max-over-ranks time
    out_host = out.cpu().numpy() if ws == 1 else None

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

    def wall_median(fn, reps):
        for _ in range(2):
            fn()
        ts = []
        for _ in range(reps):
            if ws > 1:
                torch.distributed.barrier()
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return float(np.median(ts))

    e2e_per = wall_median(e2e_call, max(3, min(args.steps, 20)))
    if ws > 1:
        tt = torch.tensor([e2e_per], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_per = float(tt.item())
    e2e_bytes = 8 * h_in.numel()
    e2e_numpy = None
    if ws == 1:
        vnp = prob.v.copy()
        t_np = wall_median(lambda: op.apply(vnp), 5)
        e2e_numpy = {"value": n / t_np * 1e-9, "unit": "GDoF/s", "ms": t_np * 1e3,
                     "path": "PhaseFieldOperator.apply(numpy float64) -> numpy (pageable copies, "
                             "what the reference driver feeds)"}

    hbm, peak_kind = peaks()
    # -------------------------------------------------------------- solve
    solve = None
    x_solve = None
    if not args.no_solve and ws == 1:
        solve, x_solve = measure_solve(prob, mask, hbm)
    elif not args.no_solve and ws > 1:
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

        try:                             # never lose the headline vmult line to the solve
            newton_step()
            setup_s, gmres_s, its = newton_step()
        except Exception as e:
            setup_s = None
            solve = {"error": f"{type(e).__name__}: {e}"[:300]}
        if setup_s is not None:
            solve = {"setup_ms": setup_s * 1e3, "gmres_ms": gmres_s * 1e3, "gmres_iters": its,
                     "ms_per_newton_step": (setup_s + gmres_s) * 1e3,
                     "rhs": "Newton RHS -A(U) from the GPU residual kernel on each slab, constrained rows zeroed",
                     "control": "slab-distributed GMRES(30) rel 1e-8 abs 0, V(1,1) FULL, Chebyshev deg %d, "
                                "%s halos + all-reduced dots" % (prob.degree, args.backend),
                     "timing": "wall clock, max over ranks"}

    strong = None
    if ws > 1 and args.strong:
        try:
            strong = measure_strong(args.strong, ws, rank, args)
        except Exception as e:          # never lose the headline line to the sub-result
            strong = {"config": args.strong, "error": f"{type(e).__name__}: {e}"[:300]}

    extra = {}
    if ws == 1 and args.extra:
        for name in [c for c in args.extra.split(",") if c and c != args.config]:
            extra[name] = measure_config(name, hbm)

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return 0

    b_c, b_f = algorithmic_bytes(prob.dim, mesh.n_vertices, mesh.n_cells,
                                 9 if getattr(mesh, "order", 1) == 2 else None)
    prof_name, pj, fresh = profile_for(args.config)
    traffic = flops = None
    if pj and fresh and ws == 1:
        traffic = pj.get("dram_bytes_per_launch")
        flops = pj.get("fp64_flops_per_launch")
    achieved = b_c / per * 1e-9
    peak_all = hbm * ws                           # aggregate over the ranks
    line = {
        "metric": METRIC, "value": value, "unit": "GDoF/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak" if (ws == 1 or args.config == "cfg2") else "strong", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded state/vector, SURVEY §8d; random-init, no dataset)",
        "config": config_dict(args, ws, prob, mesh),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak_all, "unit": "GB/s",
                     "frac": achieved / peak_all, "traffic": traffic,
                     "bytes_model": "B_C = 16 n_c V + 8 Q (2 + d(d+1)/2) C + n_c V (SURVEY §8d)",
                     "algorithmic_bytes_BC": b_c, "algorithmic_bytes_BF": b_f,
                     "frac_BF": b_f / per * 1e-9 / peak_all,
                     "frac_ncu": (traffic / per * 1e-9 / hbm) if traffic else None,
                     "profile": {"file": prof_name, "src_sha": src_sha(),
                                 "matches_current_sources": bool(fresh),
                                 "traffic_def": (pj or {}).get("traffic_def")},
                     "peak_kind": peak_kind + (f" x{ws} GPUs" if ws > 1 else ""),
                     # the kernel recomputes the coefficient tables: its own ceiling is FP64
                     # issue; flops = SASS DFMA x2 + DADD + DMUL of the ncu capture
                     "fp64": ({"achieved": flops / per * 1e-12, "peak": FP64_PEAK_TFLOPS,
                               "unit": "TFLOP/s", "frac": flops / per * 1e-12 / FP64_PEAK_TFLOPS,
                               "flops_per_launch": flops,
                               "peak_kind": "measured, tools/microbench.cu DFMA chains"}
                              if flops else None)},
        "e2e": {"value": n / e2e_per * 1e-9, "unit": "GDoF/s", "h2d_bytes_per_step": e2e_bytes,
                "d2h_bytes_per_step": e2e_bytes,
                "path": ("PhaseFieldOperator.apply(pinned host tensor, out=pinned host tensor)" if ws == 1
                         else "per rank: pinned H2D of the slab, halo exchange + vmult, D2H; bytes per rank"),
                "numpy": e2e_numpy},
        # our kernels per step: the fused vmult; on a slab (N > 1) the interior rows
        # and, after the halo lands, the two boundary rows
        "gpu_launches": args.steps * (1 if ws == 1 else (3 if getattr(mesh, "order", 1) == 2 else 2)),
        "solve": solve,
        "configs": extra or None,
        "strong_scaling": strong,
        "wall_s_timed_region": wall,
        "step_ms_min_max": [float(np.min(step_ms)), float(np.max(step_ms))],
    }
    line["clocks"] = clk.summary()
    parity = {}
    if not args.no_cpu and ws == 1:
        threads = os.cpu_count() or 1
        arm = CpuArm(prob)
        ref_out, ts, t_cache = arm.vmult(threads, 3)
        med = float(np.median(ts))
        line["cpu_baseline"] = {"value": n / med * 1e-9, "unit": "GDoF/s", "cores": threads, "kind": arm.kind,
                                "sample": f"{args.config} full-size vmult, median of 3 ({arm.what}, "
                                          f"PhaseFieldOperator.apply, model.py:368-375, {threads} threads, "
                                          f"{med * 1e3:.0f} ms each; cache build {t_cache:.2f}s excluded)",
                                "cpu_model": cpu_model()}
        parity["vmult_rel_err"] = float(np.linalg.norm(out_host - ref_out) / np.linalg.norm(ref_out))
        parity["vmult_ref"] = f"{arm.what}, same seeded vector, {args.config} full size"
    g = golden_full(args.config) if ws == 1 else None
    if solve is not None and ws == 1:
        parity["gmres_iters"] = solve["gmres_iters"]
        parity["gmres_iters_ref"] = int(g["gmres_iters"]) if g is not None else None
        parity["gmres_x_fingerprint_err"] = fingerprint_err(x_solve.cpu().numpy(), g, "gmres_x") \
            if x_solve is not None else None
        parity["ref_source"] = "tests/golden/configs_full.npz (reference fracmg, same seeded problem)"
    line["parity"] = parity or None
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    if os.environ.get("PFFMG_BENCH_WATCHDOG"):      # debugging aid: dump every thread's stack after N seconds
        import faulthandler
        faulthandler.dump_traceback_later(int(os.environ["PFFMG_BENCH_WATCHDOG"]), exit=False)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="pffmg", choices=["pffmg", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--extra", default="cfg3,cfg4,cfg5",
                    help="other configs measured as sub-results at N=1 (vmult + Newton step)")
    ap.add_argument("--strong", default="cfg5",
                    help="N > 1: the config of the strong-scaling sub-result ('' to skip)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: host-staged communication, for functional runs of N>1 on one GPU")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())

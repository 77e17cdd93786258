"""Drop-in twin of reference krylov.py on the GPU.

`gmres(op, precond, b, control=None, x0=None)` is the right-preconditioned
restarted GMRES of reference krylov.py:50-136 with identical control flow:
modified Gram-Schmidt with the conditional second pass, Givens rotations,
back substitution, true residual per restart and the same tolerance logic.
The Krylov basis V, the preconditioned directions Z and all BLAS-1 work live
on the device (libpffmg `pffmg_arnoldi_mgs`, `pffmg_multi_axpy`, deterministic
reductions); only the (m+1) x m Hessenberg column crosses to the host each
iteration for the Givens update, exactly as the reference computes it.

`estimate_spectrum` is the Jacobi-PCG Lanczos estimator of krylov.py:146-198:
the probe vector is drawn on the host with numpy's PCG64 stream (bitwise the
reference's), the CG recurrence runs on the device with its scalars kept in
device memory, and the k x k tridiagonal eigenproblem is solved on the host
with numpy.linalg.eigvalsh like the reference.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .arrays import DeviceCallable, DeviceScalar, dev, empty, host, like, norm, zeros

__all__ = ["SolverControl", "SpectrumEstimate", "NoConvergence", "gmres", "estimate_spectrum"]


@dataclass
class SolverControl:
    """Reference krylov.py:27-35."""
    abs_tol: float = 1e-10
    rel_tol: float = 1e-4
    max_iters: int = 1000
    restart: int = 30

    def tolerance(self, r0_norm):
        return max(self.abs_tol, self.rel_tol * r0_norm)


class NoConvergence(RuntimeError):
    """Reference krylov.py:38-47: carries the best iterate."""

    def __init__(self, x, residual_norm, iterations):
        super().__init__(f"no convergence after {iterations} iterations "
                         f"(residual {residual_norm:.3e})")
        self.x = x
        self.residual_norm = residual_norm
        self.iterations = iterations


# The exception class raised by gmres; patch.install() points it at the
# reference's NoConvergence so the reference's `except` clauses catch it.
_NO_CONVERGENCE = [NoConvergence]


@dataclass
class SpectrumEstimate:
    """Reference krylov.py:139-143."""
    lambda_min_hat: float
    lambda_max_hat: float
    fallback: bool = False


def _tolerance(control, r0):
    return control.tolerance(r0) if hasattr(control, "tolerance") else \
        max(control.abs_tol, control.rel_tol * r0)


class _Workspace:
    """Krylov basis storage reused across calls of the same size."""

    def __init__(self, n, m):
        self.n, self.m = n, m
        self.V = torch.zeros((m + 1, n), dtype=torch.float64, device="cuda")
        self.Z = torch.zeros((m, n), dtype=torch.float64, device="cuda")
        self.H = torch.zeros((m, m + 1), dtype=torch.float64, device="cuda")   # column j = H[:, j]
        self.ctl = torch.zeros(3 + m + 1, dtype=torch.float64, device="cuda")   # pffmg_arnoldi_mgs scratch
        self.r = torch.empty(n, dtype=torch.float64, device="cuda")
        self.y = torch.zeros(m, dtype=torch.float64, device="cuda")
        self.hpin = torch.zeros(m + 1, dtype=torch.float64).pin_memory()
        self.event = torch.cuda.Event()


_WS = {}


def _workspace(n, m):
    ws = _WS.get((n, m))
    if ws is None:
        _WS.clear()
        ws = _WS[(n, m)] = _Workspace(n, m)
    return ws


def _into(fn, src, dst):
    """dst <- fn(src), using fn's device-native form when it has one."""
    native = getattr(fn, "_pffmg_into", None)
    if native is not None:
        native(src, dst)
        return
    dst.copy_(fn(src))


def _as_callable(fn):
    """Bound `apply` of our operator -> direct device form; others -> DeviceCallable."""
    owner = getattr(fn, "__self__", None)
    if owner is not None and hasattr(owner, "apply_dev") and getattr(fn, "__name__", "") == "apply":
        def call(v):
            out = empty(v.numel())
            owner.apply_dev(_lib.FULL, v, out)
            return out
        call._pffmg_into = lambda s, d: owner.apply_dev(_lib.FULL, s, d)
        return call
    if hasattr(fn, "_pffmg_into"):
        return fn
    wrapped = DeviceCallable(fn)
    return wrapped


def gmres(op, precond, b, control=None, x0=None):
    """Right-preconditioned GMRES(m) with MGS Arnoldi (reference krylov.py:50-136).

    Returns (x, iterations) with x of the kind of `b`; raises NoConvergence."""
    control = control or SolverControl()
    _lib.require_cuda()
    opf = _as_callable(op)
    pcf = _as_callable(precond) if precond is not None else None
    bd = dev(b)
    n = bd.numel()
    x = zeros(n) if x0 is None else dev(x0).clone()
    ws = _workspace(n, int(control.restart))
    r = ws.r
    if x0 is not None and bool(torch.any(x != 0)):
        _into(opf, x, r)
        _lib.call("pffmg_sub", _lib.ptr(bd), _lib.ptr(r), _lib.ptr(r), n, _lib.stream())
    else:
        r.copy_(bd)
    r_norm = norm(r)
    tol = _tolerance(control, r_norm)
    if r_norm <= tol:
        return like(x, b), 0

    total = 0
    while True:
        m = min(int(control.restart), int(control.max_iters) - total)
        if m <= 0:
            raise _NO_CONVERGENCE[0](like(x, b), r_norm, total)
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        V, Z = ws.V, ws.Z
        torch.div(r, r_norm, out=V[0])                  # krylov.py:72
        g[0] = r_norm
        j_used = 0
        # With a device-native preconditioner the next direction's preconditioning
        # is enqueued before the host reads this column (V[j+1] is normalised on
        # the device), so the GPU works through the host's Givens update; the
        # one speculative application after convergence is discarded.
        # (only for problems whose V-cycle is short next to the host round trip:
        # on very large levels the discarded application would cost more)
        # The speculation is also skipped when this iteration is predicted to
        # converge (residual estimate extrapolated from the last two, with a
        # 4x margin): the discarded application would be a whole V-cycle.
        speculate = pcf is not None and hasattr(pcf, "_pffmg_into") and n <= (1 << 24)
        ready = False                                    # Z[j] already enqueued
        res_prev, res_cur = None, r_norm                 # |g| before / after the last column
        for j in range(m):
            if not ready:
                if pcf is None:
                    Z[j].copy_(V[j])
                else:
                    _into(pcf, V[j], Z[j])
            _into(opf, Z[j], V[j + 1])                   # w lives in V[j+1]
            total += 1
            hcol = ws.H[j]
            _lib.call("pffmg_arnoldi_mgs", _lib.ptr(V), V.stride(0), j, _lib.ptr(V[j + 1]), n,
                      _lib.ptr(hcol), _lib.ptr(ws.ctl), _lib.stream())
            ws.hpin[:j + 2].copy_(hcol[:j + 2], non_blocking=True)
            ws.event.record()
            likely_done = res_prev is not None and res_prev > 0.0 and \
                res_cur * (res_cur / res_prev) <= 4.0 * tol
            ready = speculate and j + 1 < m and not likely_done
            if ready:
                _into(pcf, V[j + 1], Z[j + 1])
            ws.event.synchronize()
            H[:j + 2, j] = ws.hpin[:j + 2].numpy()
            breakdown = H[j + 1, j] == 0.0
            for i in range(j):                           # krylov.py:111-114
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            denom = np.hypot(H[j, j], H[j + 1, j])
            cs[j] = H[j, j] / denom
            sn[j] = H[j + 1, j] / denom
            H[j, j] = denom
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            res_prev, res_cur = res_cur, abs(g[j + 1])
            j_used = j + 1
            if abs(g[j + 1]) <= tol or breakdown:
                break
        y = np.zeros(j_used)
        for i in range(j_used - 1, -1, -1):              # krylov.py:125-127
            y[i] = (g[i] - H[i, i + 1:j_used] @ y[i + 1:]) / H[i, i]
        ws.y[:j_used].copy_(torch.from_numpy(y))
        _lib.call("pffmg_multi_axpy", _lib.ptr(Z), Z.stride(0), j_used, _lib.ptr(ws.y),
                  _lib.ptr(x), n, _lib.stream())
        _into(opf, x, r)                                 # r = b - op(x)
        _lib.call("pffmg_sub", _lib.ptr(bd), _lib.ptr(r), _lib.ptr(r), n, _lib.stream())
        r_norm = norm(r)
        if r_norm <= tol * (1.0 + 1e-8):
            return like(x, b), total
        if total >= control.max_iters:
            raise _NO_CONVERGENCE[0](like(x, b), r_norm, total)


# ----------------------------------------------------------------- spectrum

_PROBES = {}


def probe_vector(seed, n):
    """numpy PCG64 standard normals (krylov.py:158-159), cached on the device."""
    key = (int(seed), int(n))
    t = _PROBES.get(key)
    if t is None:
        t = dev(np.random.default_rng(seed).standard_normal(n))
        _PROBES[key] = t
    return t


CG_MAXIT = 64


def lanczos_extremes(scal_host, n_iters):
    """Lanczos tridiagonal from CG alpha/beta -> extreme eigenvalues (krylov.py:187-198)."""
    k = int(scal_host[4])
    alphas = list(scal_host[8:8 + k])
    betas = list(scal_host[8 + CG_MAXIT:8 + CG_MAXIT + int(scal_host[5])])
    if k < 2:
        return SpectrumEstimate(1.0, 1.0, fallback=True)
    T = np.zeros((k, k))
    T[0, 0] = 1.0 / alphas[0]
    for i in range(1, k):
        T[i, i] = 1.0 / alphas[i] + betas[i - 1] / alphas[i - 1]
        off = np.sqrt(betas[i - 1]) / alphas[i - 1]
        T[i, i - 1] = off
        T[i - 1, i] = off
    ev = np.linalg.eigvalsh(T)
    return SpectrumEstimate(float(ev[0]), float(ev[-1]), fallback=False)


def lanczos_extremes_batch(scal_rows, n_iters):
    """lanczos_extremes of many CG runs at once: the tridiagonals of equal size
    go through one batched eigvalsh (numpy loops LAPACK over the stack, so every
    result equals the one-by-one call); the T entries use the same formulas."""
    rows = np.asarray(scal_rows, dtype=np.float64)
    out = [None] * len(rows)
    groups = {}
    for i, r in enumerate(rows):
        k = int(r[4])
        if k < 2:
            out[i] = SpectrumEstimate(1.0, 1.0, fallback=True)
        else:
            groups.setdefault(k, []).append(i)
    for k, idx in groups.items():
        a = rows[idx][:, 8:8 + k]
        b = rows[idx][:, 8 + CG_MAXIT:8 + CG_MAXIT + k - 1]
        T = np.zeros((len(idx), k, k))
        T[:, 0, 0] = 1.0 / a[:, 0]
        for i in range(1, k):
            T[:, i, i] = 1.0 / a[:, i] + b[:, i - 1] / a[:, i - 1]
            off = np.sqrt(b[:, i - 1]) / a[:, i - 1]
            T[:, i, i - 1] = off
            T[:, i - 1, i] = off
        ev = np.linalg.eigvalsh(T)
        for j, i in enumerate(idx):
            out[i] = SpectrumEstimate(float(ev[j, 0]), float(ev[j, -1]), fallback=False)
    return out


def cg_lanczos_dev(apply_into, diag, b, n_iters, keep_host=True):
    """Device Jacobi-PCG; apply_into(src, dst) computes dst = A src."""
    if n_iters > CG_MAXIT:
        raise ValueError(f"n_iters <= {CG_MAXIT} supported")
    n = b.numel()
    r, z, p, Ap = empty(n), empty(n), empty(n), empty(n)
    scal = torch.zeros(8 + 2 * CG_MAXIT, dtype=torch.float64, device="cuda")
    s = _lib.stream()
    _lib.call("pffmg_cg_start", _lib.ptr(b), _lib.ptr(diag), _lib.ptr(r), _lib.ptr(z),
              _lib.ptr(p), n, _lib.ptr(scal), s)
    for _ in range(n_iters):
        apply_into(p, Ap)
        for phase in range(3):
            _lib.call("pffmg_cg_step", _lib.ptr(Ap), _lib.ptr(diag), _lib.ptr(r), _lib.ptr(z),
                      _lib.ptr(p), n, _lib.ptr(scal), phase, s)
    return scal


def estimate_spectrum(op, diag_precond, n_iters=10, seed=0, constrained=None):
    """Extreme eigenvalues of D^-1 A from Jacobi-PCG (reference krylov.py:146-198)."""
    _lib.require_cuda()
    diag = dev(diag_precond)
    n = diag.numel()
    b = probe_vector(seed, n).clone()
    if constrained is not None:
        c = dev(constrained, torch.bool) if not isinstance(constrained, torch.Tensor) else constrained
        b[c.to("cuda")] = 0.0
    f = _as_callable(op)
    scal = cg_lanczos_dev(lambda src, dst: _into(f, src, dst), diag, b, n_iters)
    return lanczos_extremes(host(scal), n_iters)

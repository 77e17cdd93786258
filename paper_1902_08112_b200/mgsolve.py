"""Drop-in twin of reference mgsolve.py: GMG V-cycle preconditioner on the GPU.

Same names and signatures as reference mgsolve.py:41-283.  Two execution
paths share one control flow:

* native -- every level operator is our PhaseFieldOperator: all vectors are
  device-resident per-level buffers, each Chebyshev step is ONE fused kernel
  (block vmult + recurrence, libpffmg pffmg_cheb_step), the V-cycle residual
  is one fused kernel (pffmg_residual), transfers carry the coarse/fine
  constraint masks inside the stencil kernels, and the whole cycle is
  captured once into a CUDA graph and replayed.
* generic -- any operator implementing the reference block protocol (the
  reference's own test operators): the same algorithm driven through the
  protocol, with device BLAS-1 kernels for the vector recurrences.

Level contexts for the fracture operator (`build_level_contexts`) are built
on the device: masks and states travel to coarser levels by injection
kernels (bit-exact), diagonals by the diagonal kernel, and block spectra by
the device CG-Lanczos estimator with the reference's seed rule.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _lib
from .arrays import DeviceCallable, dev, empty, flags_buffer, host, is_tensor, like, pack_flags, zeros
from .fem import Discretization
from .krylov import cg_lanczos_dev, estimate_spectrum, lanczos_extremes, probe_vector
from .model import DeviceMask, LinearizationState, PhaseFieldOperator

__all__ = ["ChebyshevMode", "ChebyshevParams", "PreconditionerKind", "LevelContext",
           "smoother_params", "solver_params", "chebyshev_apply", "chebyshev_solver_degree",
           "build_level_contexts", "contexts_from_operators", "vcycle", "coarse_solve"]


class ChebyshevMode(Enum):
    SMOOTHER = "smoother"
    SOLVER = "solver"


class PreconditionerKind(Enum):
    FULL = "full"
    BLOCK_DIAG = "blockdiag"


@dataclass
class ChebyshevParams:
    degree: int
    a: float
    b: float
    mode: ChebyshevMode


def smoother_params(spectrum, degree=4):
    """[1.2 lmax / 5, 1.2 lmax] (mgsolve.py:59-62)."""
    top = 1.2 * spectrum.lambda_max_hat
    return ChebyshevParams(degree, top / 5.0, top, ChebyshevMode.SMOOTHER)


def solver_params(spectrum, degree):
    """[0.9 lmin, 1.2 lmax] (mgsolve.py:65-68)."""
    return ChebyshevParams(degree, 0.9 * spectrum.lambda_min_hat,
                           1.2 * spectrum.lambda_max_hat, ChebyshevMode.SOLVER)


def chebyshev_solver_degree(spectrum, target=1e-3, cap=30):
    """mgsolve.py:71-79."""
    a = 0.9 * spectrum.lambda_min_hat
    b = 1.2 * spectrum.lambda_max_hat
    if b - a <= 1e-14 * max(b, 1.0):
        return 1
    sigma = (b + a) / (b - a)
    d = int(np.ceil(np.arccosh(1.0 / target) / np.arccosh(sigma)))
    return max(1, min(cap, d))


def _cheb_coeffs(params):
    theta = 0.5 * (params.b + params.a)
    delta = 0.5 * (params.b - params.a)
    degenerate = delta <= 1e-14 * max(abs(theta), 1.0)
    return theta, delta, degenerate


# ------------------------------------------------------------ generic path

def chebyshev_apply(apply_fn, diag, params, x, b):
    """Chebyshev-accelerated Jacobi for A x = b (mgsolve.py:82-113) on the device.

    Returns the updated iterate (same kind as `x`)."""
    _lib.require_cuda()
    f = apply_fn if hasattr(apply_fn, "_pffmg_into") else DeviceCallable(apply_fn)
    inv = torch.reciprocal(dev(diag))
    xd = dev(x).clone()
    bd = dev(b)
    out = _cheb_generic(f, inv, params, xd, bd, x_is_zero=not bool(torch.any(xd != 0)))
    return like(out, x)


def _cheb_generic(f, inv, params, x, b, x_is_zero):
    n = x.numel()
    s = _lib.stream()
    theta, delta, degenerate = _cheb_coeffs(params)
    r = b.clone() if x_is_zero else b - f(x)
    if degenerate:
        for _ in range(params.degree):
            _lib.call("pffmg_jacobi_update", _lib.ptr(r), _lib.ptr(inv), theta, _lib.ptr(x), n, s)
            r = b - f(x)
        return x
    sigma = theta / delta
    rho_old = 1.0 / sigma
    d = (inv * r) / theta
    x += d
    for _ in range(params.degree - 1):
        r = r - f(d)
        rho = 1.0 / (2.0 * sigma - rho_old)
        d = (rho * rho_old) * d + (2.0 * rho / delta) * (inv * r)
        x += d
        rho_old = rho
    return x


class LevelContext:
    """Per-level solver state (mgsolve.py:116-125).  `diag` / `constrained`
    are numpy views materialised lazily; `diag_dev` / `flags` stay on the GPU."""

    def __init__(self, level, op, diag, spectra, constrained, disc, flags=None):
        self.level = level
        self.op = op
        self.spectra = spectra
        self.disc = disc
        self._diag = diag
        self._constrained = constrained
        self.flags = flags
        self.diag_dev = dev(diag) if diag is not None else None
        self.inv_dev = torch.reciprocal(self.diag_dev) if diag is not None else None

    @property
    def diag(self):
        if is_tensor(self._diag):
            self._diag = host(self._diag)
        return self._diag

    @property
    def constrained(self):
        if self._constrained is None:
            self._constrained = self.op.mask.is_constrained
        if is_tensor(self._constrained):
            self._constrained = host(self._constrained)
        return self._constrained


def _is_native(op):
    return isinstance(op, PhaseFieldOperator)


def _cg_native(op, diag_dev, eig_iters, seed):
    """Enqueue the device CG-Lanczos of both blocks (no host sync); returns the
    device scalar arrays.  Seed rule seed + 31*level + 7*k (mgsolve.py:135-136)."""
    level = getattr(getattr(op, "space", None), "level", None)
    out = []
    for k, blk in enumerate(op.blocks):
        sd = seed + 31 * level + 7 * k if level is not None else seed + 7 * k
        n = blk.stop - blk.start
        b = probe_vector(sd, n).clone()
        comp0 = 0 if k == 0 else op.dim
        ncomp = op.dim if k == 0 else 1
        _lib.call("pffmg_masked_copy", _lib.ptr(op.flags), op.V, comp0, ncomp, _lib.ptr(b),
                  _lib.ptr(b), _lib.stream())
        out.append(cg_lanczos_dev(lambda s_, d_, k=k: op.apply_dev(k, s_, d_, pre=True), diag_dev[blk],
                                  b, eig_iters))
    return out


def _estimate_blocks(op, diag_dev, eig_iters, seed):
    """Block spectra with the seed rule seed + 31*level + 7*k (mgsolve.py:128-139)."""
    spectra = []
    level = getattr(getattr(op, "space", None), "level", None)
    if _is_native(op):
        scals = host(torch.stack(_cg_native(op, diag_dev, eig_iters, seed)))
        return tuple(lanczos_extremes(s, eig_iters) for s in scals)
    for k, blk in enumerate(op.blocks):
        sd = seed + 31 * level + 7 * k if level is not None else seed + 7 * k
        if False:
            pass
        else:
            spectra.append(estimate_spectrum(lambda vb, k=k: op.apply_block(k, vb),
                                             diag_dev[blk], n_iters=eig_iters, seed=sd,
                                             constrained=np.asarray(op.mask.is_constrained)[blk]))
    return tuple(spectra)


def contexts_from_operators(disc, ops, eig_iters=10, seed=0):
    """Level contexts for arbitrary block-protocol operators (mgsolve.py:142-151)."""
    contexts = []
    for l, op in enumerate(ops):
        diag = dev(op.diagonal())
        spectra = _estimate_blocks(op, diag, eig_iters, seed)
        flags = op.flags if _is_native(op) else None
        contexts.append(LevelContext(l, op, diag, spectra,
                                     None if _is_native(op) else op.mask.is_constrained,
                                     disc, flags))
    return contexts


def build_level_contexts(disc, state, active_mask, dirichlet_mask, params, split,
                         eig_iters=10, seed=0, threads=1):
    """Phase-field level contexts from finest-level data (mgsolve.py:154-197), on the GPU."""
    _lib.require_cuda()
    D = Discretization.wrap(disc)
    hier = D.hierarchy
    L = hier.n_levels
    dim = hier.dim
    nc = dim + 1
    Vs = [m.n_vertices for m in hier.levels]
    # fine mask = Dirichlet | active, values = Dirichlet inhomogeneity (mgsolve.py:168-171)
    dir_c = dirichlet_mask.is_constrained
    if is_tensor(dir_c) or is_tensor(active_mask):
        fine_bool = dev(dir_c, torch.bool) | dev(active_mask, torch.bool)
        fine_vals = None
    else:
        fine_bool = np.asarray(dir_c, dtype=bool) | np.asarray(active_mask, dtype=bool)
        fine_vals = np.where(dir_c, dirichlet_mask.inhomogeneity, 0.0)
    flags = [None] * L
    flags[-1] = pack_flags(fine_bool, nc, Vs[-1])
    U = [None] * L
    P1 = [None] * L
    P2 = [None] * L
    PT = [None] * L
    U[-1], P1[-1], P2[-1], PT[-1] = (dev(state.U), dev(state.U_prev1), dev(state.U_prev2),
                                     dev(state.phi_tilde))
    for l in range(L - 2, -1, -1):                      # mgsolve.py:173-186
        flags[l] = flags_buffer(Vs[l])
        D.inject_flags_dev(flags[l + 1], flags[l], l)
        U[l], P1[l], P2[l] = (empty(nc * Vs[l]) for _ in range(3))
        PT[l] = empty(Vs[l])
        D.inject_dev(U[l + 1], U[l], l, nc)
        D.inject_dev(P1[l + 1], P1[l], l, nc)
        D.inject_dev(P2[l + 1], P2[l], l, nc)
        D.inject_dev(PT[l + 1], PT[l], l, 1)
    ops, diags, scals = [], [], []
    for l in range(L):
        st = LinearizationState(U=U[l], U_prev1=P1[l], U_prev2=P2[l], t=state.t,
                                t_prev1=state.t_prev1, t_prev2=state.t_prev2, phi_tilde=PT[l])
        mask = DeviceMask(flags[l], nc, Vs[l], fine_vals if l == L - 1 else None)
        if l == L - 1 and not is_tensor(fine_bool):
            mask._host = fine_bool
        op = PhaseFieldOperator(D.spaces[l], st, mask, params, split, threads, _flags=flags[l])
        diag = empty(op.n_dofs)
        op.diagonal_dev(diag)
        ops.append(op)
        diags.append(diag)
        scals += _cg_native(op, diag, eig_iters, seed)        # enqueued, no host sync
    scal_host = host(torch.stack(scals))                      # one sync for all levels
    contexts = []
    for l in range(L):
        spectra = tuple(lanczos_extremes(scal_host[2 * l + k], eig_iters) for k in range(2))
        contexts.append(LevelContext(l, ops[l], diags[l], spectra, None, disc, flags[l]))
    return contexts


# ------------------------------------------------------------- V-cycle

def _kind_value(kind):
    return getattr(kind, "value", kind)


def coarse_solve(ctx, r, target=1e-3, cap=30):
    """Blockwise Chebyshev solve on the coarsest level (mgsolve.py:209-218)."""
    rd = dev(r)
    if _is_native(ctx.op):
        cyc = _NativeCycle.get([ctx], 4, target, cap)
        out = empty(rd.numel())
        cyc.coarse(rd, out)
        return like(out, r)
    x = zeros(rd.numel())
    f_ops = _block_callables(ctx)
    for k, blk in enumerate(ctx.op.blocks):
        degree = chebyshev_solver_degree(ctx.spectra[k], target, cap)
        prm = solver_params(ctx.spectra[k], degree)
        x[blk] = _cheb_generic(f_ops[k], ctx.inv_dev[blk], prm, x[blk].clone(), rd[blk].clone(), True)
    return like(x, r)


def _block_callables(ctx):
    return [DeviceCallable(lambda vb, k=k: ctx.op.apply_block(k, vb)) for k in range(2)]


def vcycle(contexts, kind, r, degree=4, coarse_target=1e-3, coarse_cap=30):
    """One V(1,1) cycle on a fine-level residual (mgsolve.py:262-283)."""
    _lib.require_cuda()
    rd = dev(r)
    if all(_is_native(c.op) for c in contexts):
        cyc = _NativeCycle.get(contexts, degree, coarse_target, coarse_cap)
        out = empty(rd.numel())
        cyc.run(_kind_value(kind), rd, out)
        return like(out, r)
    return like(_generic_vcycle(contexts, _kind_value(kind), rd, degree, coarse_target, coarse_cap), r)


def _generic_vcycle(contexts, kind, r, degree, target, cap):
    fine = contexts[-1]
    r = r.clone()
    cons = [dev(c.constrained, torch.bool) for c in contexts]
    r[cons[-1]] = 0.0
    top = len(contexts) - 1
    D = Discretization.wrap(fine.disc)
    if kind == "full":
        return _gen_mono(contexts, cons, D, r, top, degree, target, cap)
    dim = D.dim
    out = torch.zeros_like(r)
    for k, blk in enumerate(fine.op.blocks):
        out[blk] = _gen_block(contexts, cons, D, k, r[blk].clone(), top, degree, target, cap,
                              dim if k == 0 else 1)
    return out


def _gen_smooth(ctx, x, b, degree):
    f = _block_callables(ctx)
    for k, blk in enumerate(ctx.op.blocks):
        prm = smoother_params(ctx.spectra[k], degree)
        xb = x[blk].clone()
        x[blk] = _cheb_generic(f[k], ctx.inv_dev[blk], prm, xb, b[blk].clone(),
                               not bool(torch.any(xb != 0)))
    return x


def _gen_mono(ctxs, cons, D, r, l, degree, target, cap):
    ctx = ctxs[l]
    if l == 0:
        return dev(coarse_solve(ctx, r, target, cap))
    x = _gen_smooth(ctx, torch.zeros_like(r), r, degree)
    d = r - DeviceCallable(ctx.op.apply)(x)
    rc = D.restrict(d, l - 1)
    rc[cons[l - 1]] = 0.0
    ec = _gen_mono(ctxs, cons, D, rc, l - 1, degree, target, cap)
    ef = D.prolongate(ec, l - 1)
    ef[cons[l]] = 0.0
    x += ef
    return _gen_smooth(ctx, x, r, degree)


def _gen_block(ctxs, cons, D, k, rb, l, degree, target, cap, n_comp):
    ctx = ctxs[l]
    blk = ctx.op.blocks[k]
    f = _block_callables(ctx)[k]
    inv = ctx.inv_dev[blk]
    if l == 0:
        deg = chebyshev_solver_degree(ctx.spectra[k], target, cap)
        return _cheb_generic(f, inv, solver_params(ctx.spectra[k], deg), torch.zeros_like(rb), rb, True)
    prm = smoother_params(ctx.spectra[k], degree)
    x = _cheb_generic(f, inv, prm, torch.zeros_like(rb), rb, True)
    d = rb - f(x)
    rc = D.restrict_block(d, l - 1, n_comp)
    rc[cons[l - 1][ctxs[l - 1].op.blocks[k]]] = 0.0
    ec = _gen_block(ctxs, cons, D, k, rc, l - 1, degree, target, cap, n_comp)
    ef = D.prolongate_block(ec, l - 1, n_comp)
    ef[cons[l][blk]] = 0.0
    x += ef
    return _cheb_generic(f, inv, prm, x, rb, not bool(torch.any(x != 0)))


# ---------------------------------------------------------- native V-cycle

class _Level:
    """Device buffers of one level for the native cycle."""

    def __init__(self, ctx):
        op = ctx.op
        self.ctx = ctx
        self.op = op
        self.n = op.n_dofs
        self.dim = op.dim
        self.V = op.V
        self.flags = op.flags
        self.inv = ctx.inv_dev
        n = self.n
        self.r = zeros(n)       # right-hand side of this level
        self.x = zeros(n)       # iterate / correction
        self.res = zeros(n)     # V-cycle residual d = r - A x
        self.cr = zeros(n)      # Chebyshev residual
        self.d0 = zeros(n)
        self.d1 = zeros(n)

    def blk(self, k):
        return slice(0, self.dim * self.V) if k == 0 else slice(self.dim * self.V, self.n)


class _NativeCycle:
    """V(1,1) cycle over native contexts, optionally replayed from a CUDA graph."""

    _cache = {}

    @classmethod
    def get(cls, contexts, degree, target, cap):
        key = (tuple(id(c) for c in contexts), degree, target, cap)
        hit = cls._cache.get(key)
        if hit is not None and all(a is b for a, b in zip(hit.contexts, contexts)):
            return hit
        if len(cls._cache) > 8:
            cls._cache.clear()
        cyc = cls(contexts, degree, target, cap)
        cls._cache[key] = cyc
        return cyc

    def __init__(self, contexts, degree, target, cap):
        self.contexts = list(contexts)
        self.degree = degree
        self.levels = [_Level(c) for c in contexts]
        self.disc = Discretization.wrap(contexts[-1].disc) if len(contexts) > 1 else None
        self.smooth_prm = [[smoother_params(c.spectra[k], degree) for k in range(2)] for c in contexts]
        self.coarse_prm = [solver_params(contexts[0].spectra[k],
                                         chebyshev_solver_degree(contexts[0].spectra[k], target, cap))
                           for k in range(2)]
        self.use_graph = os.environ.get("PFFMG_GRAPHS", "1") != "0"
        self.graphs = {}
        self.r_in = None
        self.x_out = None

    # one Chebyshev sweep on block k of level L: x (zero or not) -> smoothed x
    def _cheb(self, L, k, prm, x_is_zero, pre=True):
        op = L.op
        b = L.blk(k)
        x, r, rhs, inv = L.x[b], L.cr[b], L.r[b], L.inv[b]
        d_in, d_out = L.d0[b], L.d1[b]
        nb = x.numel()
        s = _lib.stream()
        theta, delta, degenerate = _cheb_coeffs(prm)
        if degenerate:                                     # mgsolve.py:97-101
            if x_is_zero:
                x.zero_()
                r.copy_(rhs)
            else:
                op.residual_dev(k, x, rhs, r, pre=pre)
            for _ in range(prm.degree):
                _lib.call("pffmg_jacobi_update", _lib.ptr(r), _lib.ptr(inv), theta, _lib.ptr(x), nb, s)
                op.residual_dev(k, x, rhs, r, pre=pre)
            return
        sigma = theta / delta
        rho_old = 1.0 / sigma
        if x_is_zero:                                      # r = b; d = inv r / theta; x = d
            _lib.call("pffmg_cheb_init_zero", _lib.ptr(rhs), _lib.ptr(inv), theta, _lib.ptr(r),
                      _lib.ptr(d_in), _lib.ptr(x), nb, s)
            pending = False
        else:                                              # r = b - A x; d = inv r / theta
            op.cheb_init_dev(k, x, rhs, r, d_in, inv, theta, pre=pre)
            pending = True                                 # x += d folded into the next step
        for _ in range(prm.degree - 1):
            rho = 1.0 / (2.0 * sigma - rho_old)
            op.cheb_step_dev(k, d_in, d_out, r, x, inv, rho * rho_old, 2.0 * rho / delta, pending,
                             pre=pre)
            pending = False
            d_in, d_out = d_out, d_in
            rho_old = rho
        if pending:                                        # degree 1 from a non-zero x
            _lib.call("pffmg_axpy", 1.0, _lib.ptr(d_in), _lib.ptr(x), nb, s)

    def _smooth(self, l, x_is_zero):
        L = self.levels[l]
        for k in range(2):
            self._cheb(L, k, self.smooth_prm[l][k], x_is_zero)

    def _coarse_into_x(self, pre=True):
        L = self.levels[0]
        for k in range(2):
            self._cheb(L, k, self.coarse_prm[k], True, pre)

    def _cycle(self, l):                                   # mgsolve.py:221-235
        if l == 0:
            self._coarse_into_x()
            return
        L, Lc = self.levels[l], self.levels[l - 1]
        self._smooth(l, True)
        L.op.residual_dev(_lib.FULL, L.x, L.r, L.res, pre=True)
        self.disc.restrict_dev(L.res, Lc.r, l - 1, L.dim + 1, 0, Lc.flags)
        self._cycle(l - 1)
        self.disc.prolongate_dev(Lc.x, L.x, l - 1, L.dim + 1, 0, L.flags, accumulate=True)
        self._smooth(l, False)

    def _block_cycle(self, k, l):                          # mgsolve.py:238-259
        L = self.levels[l]
        if l == 0:
            self._cheb(L, k, self.coarse_prm[k], True)
            return
        Lc = self.levels[l - 1]
        b = L.blk(k)
        self._cheb(L, k, self.smooth_prm[l][k], True)
        L.op.residual_dev(k, L.x[b], L.r[b], L.res[b], pre=True)
        ncomp = L.dim if k == 0 else 1
        comp0 = 0 if k == 0 else L.dim
        self.disc.restrict_dev(L.res[b], Lc.r[Lc.blk(k)], l - 1, ncomp, comp0, Lc.flags)
        self._block_cycle(k, l - 1)
        self.disc.prolongate_dev(Lc.x[Lc.blk(k)], L.x[b], l - 1, ncomp, comp0, L.flags,
                                 accumulate=True)
        self._cheb(L, k, self.smooth_prm[l][k], False)

    def _body(self, kind):
        top = self.levels[-1]
        _lib.call("pffmg_masked_copy", _lib.ptr(top.flags), top.V, 0, top.dim + 1,
                  _lib.ptr(self.r_in), _lib.ptr(top.r), _lib.stream())    # r[constrained] = 0
        if kind == "full":
            self._cycle(len(self.levels) - 1)
        else:
            for k in range(2):
                self._block_cycle(k, len(self.levels) - 1)
        self.x_out.copy_(top.x)

    def run(self, kind, r, out):
        top = self.levels[-1]
        if self.r_in is None:
            self.r_in = zeros(top.n)
            self.x_out = zeros(top.n)
        self.r_in.copy_(r)
        if self.use_graph:
            g = self.graphs.get(kind)
            if g is None:
                self._body(kind)                       # warm-up (allocator, lazy attributes)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._body(kind)
                self.graphs[kind] = g
            g.replay()
        else:
            self._body(kind)
        out.copy_(self.x_out)

    def coarse(self, r, out):
        """Public coarse_solve: r is arbitrary (not masked), so no pre-mask hint."""
        L = self.levels[0]
        L.r.copy_(r)
        self._coarse_into_x(pre=False)
        out.copy_(L.x)


class VCyclePreconditioner:
    """Callable precond for gmres that writes straight into the Krylov slot."""

    def __init__(self, contexts, kind=PreconditionerKind.FULL, degree=4, coarse_target=1e-3,
                 coarse_cap=30):
        self.contexts = contexts
        self.kind = _kind_value(kind)
        self.cycle = _NativeCycle.get(contexts, degree, coarse_target, coarse_cap)

    def __call__(self, r):
        rd = dev(r)
        out = empty(rd.numel())
        self.cycle.run(self.kind, rd, out)
        return like(out, r)

    def _pffmg_into(self, src, dst):
        self.cycle.run(self.kind, src, dst)

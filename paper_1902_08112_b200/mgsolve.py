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
from .arrays import DeviceCallable, copy_into, dev, empty, flags_buffer, host, is_tensor, like, pack_flags, zeros
from .fem import Discretization
from .krylov import cg_lanczos_dev, estimate_spectrum, lanczos_extremes, lanczos_extremes_batch, probe_vector
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

    def __init__(self, level, op, diag, spectra, constrained, disc, flags=None, inv=None):
        self.level = level
        self.op = op
        self.spectra = spectra
        self.disc = disc
        self._diag = diag
        self._constrained = constrained
        self.flags = flags
        self.diag_dev = dev(diag) if diag is not None else None
        if inv is not None:
            self.inv_dev = inv
        else:
            self.inv_dev = torch.reciprocal(self.diag_dev) if diag is not None else None
        self._session = None     # set by _Session.build: contexts of a reusable setup
        self._gen = 0

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


def _cg_native(op, diag_dev, eig_iters, seed, blocks=(0, 1)):
    """Enqueue the device CG-Lanczos of the given blocks (no host sync); returns the
    device scalar arrays.  Seed rule seed + 31*level + 7*k (mgsolve.py:135-136)."""
    level = getattr(getattr(op, "space", None), "level", None)
    out = []
    for k in blocks:
        blk = op.blocks[k]
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


def _fine_mask(dirichlet_mask, active_mask):
    """fine mask = Dirichlet | active, values = Dirichlet inhomogeneity (mgsolve.py:168-171).
    The union is formed on the device; the host views (numpy inputs only) are
    lazily evaluated callables -- the solve never needs them."""
    dir_c = dirichlet_mask.is_constrained
    fine_dev = dev(dir_c, torch.bool) | dev(active_mask, torch.bool)
    if is_tensor(dir_c) or is_tensor(active_mask):
        return fine_dev, None, None
    inh = dirichlet_mask.inhomogeneity

    def vals():
        return np.where(np.asarray(dir_c, dtype=bool), inh, 0.0)

    def union():
        return np.asarray(dir_c, dtype=bool) | np.asarray(active_mask, dtype=bool)
    return fine_dev, vals, union


# Reuse of the device setup across Newton steps (see _Session); PFFMG_REUSE_SETUP=0
# rebuilds every buffer and re-records every graph on each call instead.
REUSE_SETUP = os.environ.get("PFFMG_REUSE_SETUP", "1") != "0"
# Smooth both diagonal blocks with one block-diagonal kernel per Chebyshev step
# (PFFMG_BLOCKDIAG_SMOOTH=0: one kernel per block and step, the reference's order).
BLOCKDIAG_SMOOTH = os.environ.get("PFFMG_BLOCKDIAG_SMOOTH", "1") != "0"
# Coarsest-level solve in one kernel (pffmg_coarse_cheb) when the level is small;
# PFFMG_COARSE_KERNEL=0: one kernel per Chebyshev step.
COARSE_KERNEL = os.environ.get("PFFMG_COARSE_KERNEL", "1") != "0"
# Restriction into a level fused with that level's smoother start from x = 0
# (pffmg_restrict_init_bd); PFFMG_FUSED_DESCENT=0: separate kernels.
FUSED_DESCENT = os.environ.get("PFFMG_FUSED_DESCENT", "1") != "0"
# x = 0 starts store d only and the first Chebyshev step reads r from the
# right-hand side and x from d (pffmg_cheb_first_*); PFFMG_LEAN_START=0: the
# start writes r, d, x and every step is a pffmg_cheb_step_*.
LEAN_START = os.environ.get("PFFMG_LEAN_START", "1") != "0"
# The multi-stream setup (2L concurrent CG-Lanczos chains) launches with
# programmatic dependent launch (PFFMG_SETUP_PDL=0: fully stream-ordered).
SETUP_PDL = os.environ.get("PFFMG_SETUP_PDL", "1") != "0"
# block-diagonal smoothing kernel (both blocks per launch) on levels with fewer
# vertices than these; larger levels run the two block kernels per step
BD_MAXV2 = int(os.environ.get("PFFMG_BD_MAXV2", str(1 << 40)))
BD_MAXV3 = int(os.environ.get("PFFMG_BD_MAXV3", str(1 << 17)))


def build_level_contexts(disc, state, active_mask, dirichlet_mask, params, split,
                         eig_iters=10, seed=0, threads=1):
    """Phase-field level contexts from finest-level data (mgsolve.py:154-197), on the GPU."""
    _lib.require_cuda()
    D = Discretization.wrap(disc)
    fine_bool, fine_vals, fine_host = _fine_mask(dirichlet_mask, active_mask)
    if REUSE_SETUP:
        sess = _Session.get(D, params, split, state.t, eig_iters, seed, threads)
        return sess.build(disc, state, fine_bool, fine_vals, fine_host)
    return _build_fresh(disc, D, state, fine_bool, fine_vals, fine_host, params, split, eig_iters, seed,
                        threads)


def _build_fresh(disc, D, state, fine_bool, fine_vals, fine_host, params, split, eig_iters, seed, threads):
    hier = D.hierarchy
    L = hier.n_levels
    dim = hier.dim
    nc = dim + 1
    Vs = [m.n_vertices for m in hier.levels]
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
        if l == L - 1:
            mask._host_fn = fine_host
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


class _Session:
    """Device buffers, operators and recorded graphs of one hierarchy, reused by
    every build_level_contexts call with the same hierarchy / material / split.

    A Newton loop rebuilds its level contexts once per step; only the state
    values change, never the shapes.  The session keeps the per-level state,
    flag, diagonal and inverse-diagonal buffers, records the whole device
    setup (injections, diagonals, CG-Lanczos of both blocks on every level)
    as one CUDA graph, and keeps the V-cycle graphs whose Chebyshev scalars
    are read from device memory (libpffmg *_dc entry points), so a step costs
    graph replays plus one host sync for the spectra.

    Contexts keep the reference's value semantics: when a new build starts
    while contexts (or operators) of the previous build are still referenced,
    those are first detached onto private copies of their buffers."""

    _cache = {}
    MAX = 2

    @classmethod
    def get(cls, D, params, split, t, eig_iters, seed, threads):
        from .model import _split_code
        mf = getattr(params, "modulus_field", None)
        key = (id(D.hierarchy), _split_code(split), float(params.mu), float(params.lam),
               float(params.g_c), float(params.kappa), float(params.eps), float(params.pressure(t)),
               float(getattr(params, "split_band", 0.0) or 0.0), id(mf), int(eig_iters), int(seed))
        sess = cls._cache.get(key)
        if sess is not None and sess.hier is D.hierarchy and sess.modulus is mf:
            cls._cache[key] = cls._cache.pop(key)          # most recently used last
            return sess
        while len(cls._cache) >= cls.MAX:
            cls._cache.pop(next(iter(cls._cache)))
        sess = cls(D, params, split, t, eig_iters, seed, threads)
        cls._cache[key] = sess
        return sess

    def __init__(self, D, params, split, t, eig_iters, seed, threads):
        self.D = D
        self.hier = D.hierarchy
        self.modulus = getattr(params, "modulus_field", None)
        self.params, self.split, self.threads = params, split, threads
        self.eig_iters, self.seed = int(eig_iters), int(seed)
        L = self.L = self.hier.n_levels
        self.dim = self.hier.dim
        nc = self.nc = self.dim + 1
        Vs = self.Vs = [m.n_vertices for m in self.hier.levels]
        self.U = [zeros(nc * V) for V in Vs]
        self.P1 = [zeros(nc * V) for V in Vs]
        self.P2 = [zeros(nc * V) for V in Vs]
        self.PT = [zeros(V) for V in Vs]
        self.flags = [flags_buffer(V) for V in Vs]
        self.diag = [zeros(nc * V) for V in Vs]
        self.inv = [zeros(nc * V) for V in Vs]
        self.ops = []
        for l in range(L):
            st = LinearizationState(U=self.U[l], U_prev1=self.P1[l], U_prev2=self.P2[l], t=t,
                                    t_prev1=t, t_prev2=t, phi_tilde=self.PT[l])
            self.ops.append(PhaseFieldOperator(D.spaces[l], st, DeviceMask(self.flags[l], nc, Vs[l]),
                                               params, split, threads, _flags=self.flags[l]))
        self.graph = None
        self.scal = None
        self.use_graph = os.environ.get("PFFMG_GRAPHS", "1") != "0"
        self.gen = 0
        self.spectra = None
        self._prev = []
        self._cycles = {}
        self._streams = None

    # -- device work of one setup (recorded once, replayed per Newton step)
    def _device_setup(self):
        """Fine level first: each level's state injection (mgsolve.py:173-186),
        phi table (_build_caches, model.py:260), diagonal and inverse diagonal go
        on the main stream, and its two block CG-Lanczos runs start on their own
        streams right after -- the fine level's chains (the critical path) no
        longer wait for the coarse levels' setup kernels.  The 2L chains are
        independent (each stream has its own reduction scratch in libpffmg)."""
        if not SETUP_PDL:
            prev = _lib.C.c_int(1)
            _lib.call("pffmg_set_pdl", 0, _lib.C.byref(prev))
            try:
                return self._device_setup_body()
            finally:
                _lib.call("pffmg_set_pdl", prev.value, None)
        return self._device_setup_body()

    def _device_setup_body(self):
        D, s = self.D, _lib.stream()
        main = torch.cuda.current_stream()
        if self._streams is None:
            self._streams = [torch.cuda.Stream() for _ in range(2 * self.L)]
        scals = [[None, None] for _ in range(self.L)]
        for l in range(self.L - 1, -1, -1):
            if l < self.L - 1:
                D.inject_flags_dev(self.flags[l + 1], self.flags[l], l)
                D.inject_dev(self.U[l + 1], self.U[l], l, self.nc)
                D.inject_dev(self.P1[l + 1], self.P1[l], l, self.nc)
                D.inject_dev(self.P2[l + 1], self.P2[l], l, self.nc)
                D.inject_dev(self.PT[l + 1], self.PT[l], l, 1)
            self.ops[l].build_phi_coef()
            self.ops[l].diagonal_dev(self.diag[l])
            _lib.call("pffmg_reciprocal", _lib.ptr(self.diag[l]), _lib.ptr(self.inv[l]),
                      self.diag[l].numel(), s)
            for k in range(2):
                st = self._streams[2 * l + k]
                st.wait_stream(main)
                with torch.cuda.stream(st):
                    scals[l][k] = _cg_native(self.ops[l], self.diag[l], self.eig_iters, self.seed, (k,))[0]
        for st in self._streams:
            main.wait_stream(st)
        return torch.stack([t for pair in scals for t in pair])

    def _detach_previous(self):
        """Give still-referenced contexts / operators of the last build private buffers."""
        prev, self._prev = self._prev, []
        for l, op_ref, ctx_ref in prev:
            op, ctx = op_ref(), ctx_ref()
            if op is None and ctx is None:
                continue
            fl = flags_buffer(self.Vs[l])
            fl.copy_(self.flags[l])
            if op is not None:
                U, P1, P2, PT = (self.U[l].clone(), self.P1[l].clone(), self.P2[l].clone(),
                                 self.PT[l].clone())
                op._rebind(U, PT, fl)
                op.state = LinearizationState(U=U, U_prev1=P1, U_prev2=P2, t=op.state.t,
                                              t_prev1=op.state.t_prev1, t_prev2=op.state.t_prev2,
                                              phi_tilde=PT)
            if ctx is not None:
                d = self.diag[l].clone()
                if ctx._diag is ctx.diag_dev:
                    ctx._diag = d
                ctx.diag_dev = d
                ctx.inv_dev = self.inv[l].clone()
                ctx.flags = fl
                ctx._session = None

    def build(self, disc, state, fine_bool, fine_vals, fine_host=None):
        import weakref
        self._detach_previous()
        L, nc = self.L, self.nc
        for buf, src in ((self.U[-1], state.U), (self.P1[-1], state.U_prev1),
                         (self.P2[-1], state.U_prev2), (self.PT[-1], state.phi_tilde)):
            copy_into(buf, src)
        m = dev(fine_bool, torch.uint8) if not is_tensor(fine_bool) else fine_bool.to(torch.uint8).contiguous()
        _lib.call("pffmg_pack_flags", _lib.ptr(m), nc, self.Vs[-1], _lib.ptr(self.flags[-1]), _lib.stream())
        if not self.use_graph:
            scal = self._device_setup()
        elif self.graph is None:
            scal = self._device_setup()                    # eager run: this build's results
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.scal = self._device_setup()
            self.graph = g
        else:
            self.graph.replay()
            scal = self.scal
        scal_host = host(scal)                             # one sync for all levels
        ei = self.eig_iters
        sp = lanczos_extremes_batch(scal_host, ei)
        self.spectra = [(sp[2 * l], sp[2 * l + 1]) for l in range(L)]
        self.gen += 1
        contexts = []
        for l in range(L):
            st = LinearizationState(U=self.U[l], U_prev1=self.P1[l], U_prev2=self.P2[l], t=state.t,
                                    t_prev1=state.t_prev1, t_prev2=state.t_prev2, phi_tilde=self.PT[l])
            mask = DeviceMask(self.flags[l], nc, self.Vs[l], fine_vals if l == L - 1 else None)
            if l == L - 1:
                mask._host_fn = fine_host
            op = PhaseFieldOperator(self.D.spaces[l], st, mask, self.params, self.split, self.threads,
                                    _flags=self.flags[l], _rho=self.ops[l]._rho, _ptab=self.ops[l]._ptab)
            ctx = LevelContext(l, op, self.diag[l], self.spectra[l], None, disc, self.flags[l],
                               inv=self.inv[l])
            ctx._session, ctx._gen = self, self.gen
            contexts.append(ctx)
            self._prev.append((l, weakref.ref(op), weakref.ref(ctx)))
        return contexts

    def owns(self, contexts):
        return (len(contexts) == self.L and
                all(getattr(c, "_session", None) is self and c._gen == self.gen for c in contexts))

    def cycle(self, degree, target, cap):
        """The session's V-cycle, coefficients of the current build."""
        key = (degree, target, cap)
        cyc = self._cycles.get(key)
        internal = [LevelContext(l, self.ops[l], self.diag[l], self.spectra[l], None, self.D,
                                 self.flags[l], inv=self.inv[l]) for l in range(self.L)]
        if cyc is None:
            cyc = _NativeCycle(internal, degree, target, cap)
            cyc.gen = self.gen
            self._cycles[key] = cyc
        elif cyc.gen != self.gen:
            cyc.set_spectra(internal)
            cyc.gen = self.gen
        return cyc


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

COARSE_SMEM_MAX = 200 * 1024


def coarse_smem_bytes(dim, ncell, V, order=1):
    """Shared-memory footprint of pffmg_coarse_cheb on a level (the formula of
    csrc/coarse.cu); levels above COARSE_SMEM_MAX run the per-step kernels."""
    nco = dim + 1
    npc = 9 if order == 2 else (1 << dim)
    maxa = 4 if order == 2 else (1 << dim)
    return 8 * (ncell * nco * npc + V * (5 * nco + 1)) + 4 * (ncell * npc + V * maxa) + V + 16


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
        # one block-diagonal kernel per Chebyshev step pays in 2D and on small
        # (launch-latency-bound) 3D levels; large 3D levels are FP64-bound and
        # run faster as two block kernels (measured, cfg4)
        self.index = ctx.level
        self.bd_ok = self.V < (BD_MAXV2 if self.dim == 2 else BD_MAXV3)
        info = op.lat.info
        self.coarse_ok = (int(np.prod(info.ncell)) <= 256 and tuple(info.own) == (0, 0)
                          and coarse_smem_bytes(self.dim, int(np.prod(info.ncell)), self.V,
                                                getattr(info, "order", 1)) <= COARSE_SMEM_MAX)

    def blk(self, k):
        return slice(0, self.dim * self.V) if k == 0 else slice(self.dim * self.V, self.n)


class _NativeCycle:
    """V(1,1) cycle over native contexts, optionally replayed from a CUDA graph."""

    _cache = {}

    @classmethod
    def get(cls, contexts, degree, target, cap):
        sess = getattr(contexts[-1], "_session", None)
        if sess is not None and sess.owns(contexts):
            return sess.cycle(degree, target, cap)
        key = (tuple(id(c) for c in contexts), degree, target, cap)
        hit = cls._cache.get(key)
        if hit is not None and all(a is b for a, b in zip(hit.contexts, contexts)):
            return hit
        if len(cls._cache) > 8:
            cls._cache.clear()
        cyc = cls(contexts, degree, target, cap)
        cls._cache[key] = cyc
        return cyc

    def __init__(self, contexts, degree, target, cap, comm=None):
        """`comm` (optional) makes the cycle slab-distributed: it provides
        halo(l, vec, n_comp) -- refresh the ghost planes of a level-l vector
        before a stencil reads it -- and restrict(l, fine, coarse, n_comp, comp0)
        / prolongate(l, coarse, fine, n_comp, comp0) between levels l and l+1
        (dist_solver.DistGMG).  Distributed cycles are not graph-recorded."""
        self.contexts = list(contexts)
        self.degree = degree
        self.comm = comm
        self.levels = [_Level(c) for c in contexts]
        self.disc = (Discretization.wrap(contexts[-1].disc) if len(contexts) > 1 and comm is None
                     else None)
        self.target, self.cap = target, cap
        self.use_graph = comm is None and os.environ.get("PFFMG_GRAPHS", "1") != "0"
        self.graphs = {}
        self.coef = None
        self.struct = None
        self.set_spectra(contexts)

    def set_spectra(self, contexts):
        """Chebyshev parameters of every (level, block) smoother and of the coarse
        solver, laid out as one device table the kernels read at run time:
        slot = [theta, c_dd_1, c_dr_1, c_dd_2, c_dr_2, ...] (mgsolve.py:97-113).
        Recorded graphs stay valid while the structure (degrees, degenerate
        branches) is unchanged; otherwise they are dropped and re-recorded."""
        self.smooth_prm = [[smoother_params(c.spectra[k], self.degree) for k in range(2)]
                           for c in contexts]
        self.coarse_prm = [solver_params(contexts[0].spectra[k],
                                         chebyshev_solver_degree(contexts[0].spectra[k], self.target,
                                                                 self.cap))
                           for k in range(2)]
        table, struct, self.slot = [], [], {}
        items = [(("s", l, k), self.smooth_prm[l][k]) for l in range(len(contexts)) for k in range(2)]
        items += [(("c", 0, k), self.coarse_prm[k]) for k in range(2)]
        for key, prm in items:
            theta, delta, degenerate = _cheb_coeffs(prm)
            self.slot[key] = (len(table), prm, degenerate)
            struct.append((key, prm.degree, degenerate))
            table.append(theta)
            if not degenerate:
                sigma = theta / delta
                rho_old = 1.0 / sigma
                for _ in range(prm.degree - 1):
                    rho = 1.0 / (2.0 * sigma - rho_old)
                    table += [rho * rho_old, 2.0 * rho / delta]
                    rho_old = rho
        table = torch.tensor(table, dtype=torch.float64)
        if self.coef is None or tuple(struct) != self.struct:
            self.coef = table.to("cuda")
            self.struct = tuple(struct)
            self.graphs = {}
        else:
            self.coef.copy_(table)

    def _halo(self, L, vec, n_comp):
        if self.comm is not None:
            self.comm.halo(L.index, vec, n_comp)

    def _stencil(self, L, vec, n_comp, call):
        """`call()` (one operator kernel on level L reading `vec`) after a
        refresh of vec's ghost planes.  Slab-distributed levels overlap the
        exchange with the interior planes (their cells read owned planes
        only) and finish the boundary planes once it has landed."""
        comm = self.comm
        plan = comm.overlap_plan(L.index) if comm is not None else None
        if plan is None:
            self._halo(L, vec, n_comp)
            call()
            return
        interior, ends = plan
        h = comm.halo_start(L.index, vec, n_comp)
        with L.op.scope(interior):
            call()
        comm.halo_finish(L.index, h)
        for sc in ends:
            with L.op.scope(sc):
                call()

    def _restrict(self, l, fine, coarse, n_comp, comp0, coarse_flags):
        if self.comm is not None:
            self.comm.restrict(l, fine, coarse, n_comp, comp0)
        else:
            self.disc.restrict_dev(fine, coarse, l, n_comp, comp0, coarse_flags)

    def _prolongate(self, l, coarse, fine, n_comp, comp0, fine_flags):
        if self.comm is not None:
            self.comm.prolongate(l, coarse, fine, n_comp, comp0)
        else:
            self.disc.prolongate_dev(coarse, fine, l, n_comp, comp0, fine_flags, accumulate=True)

    # one Chebyshev sweep on block k of level L: x (zero or not) -> smoothed x
    def _cheb(self, L, k, slot, x_is_zero, pre=True):
        op = L.op
        b = L.blk(k)
        x, r, rhs, inv = L.x[b], L.cr[b], L.r[b], L.inv[b]
        d_in, d_out = L.d0[b], L.d1[b]
        nb = x.numel()
        s = _lib.stream()
        off, prm, degenerate = self.slot[slot]
        coef = self.coef
        theta = coef[off:off + 1]
        if degenerate:                                     # mgsolve.py:97-101
            nk = L.dim if k == 0 else 1
            if x_is_zero:
                x.zero_()
                r.copy_(rhs)
            else:
                self._stencil(L, x, nk, lambda: op.residual_dev(k, x, rhs, r, pre=pre))
            for _ in range(prm.degree):
                _lib.call("pffmg_jacobi_update_dc", _lib.ptr(r), _lib.ptr(inv), _lib.ptr(theta),
                          _lib.ptr(x), nb, s)
                self._stencil(L, x, nk, lambda: op.residual_dev(k, x, rhs, r, pre=pre))
            return
        lean = x_is_zero and LEAN_START and prm.degree >= 2
        if x_is_zero:                                      # r = b; d = inv r / theta; x = d
            _lib.call("pffmg_cheb_init_zero_dc", _lib.ptr(rhs), _lib.ptr(inv), _lib.ptr(theta),
                      None if lean else _lib.ptr(r), _lib.ptr(d_in), None if lean else _lib.ptr(x), nb, s)
            pending = False
        else:                                              # r = b - A x; d = inv r / theta
            self._stencil(L, x, L.dim if k == 0 else 1,
                          lambda: op.cheb_init_dc(k, x, rhs, r, d_in, inv, theta, pre=pre))
            pending = True                                 # x += d folded into the next step
        for i in range(prm.degree - 1):
            c = coef[off + 1 + 2 * i: off + 3 + 2 * i]
            if lean and i == 0:                            # r read from rhs, x = d_in + d_out
                self._stencil(L, d_in, L.dim if k == 0 else 1,
                              lambda: op.cheb_first_dc(k, d_in, rhs, d_out, r, x, inv, c, pre=pre))
            else:
                self._stencil(L, d_in, L.dim if k == 0 else 1,
                              lambda: op.cheb_step_dc(k, d_in, d_out, r, x, inv, c, pending, pre=pre))
            pending = False
            d_in, d_out = d_out, d_in
        if pending:                                        # degree 1 from a non-zero x
            _lib.call("pffmg_axpy", 1.0, _lib.ptr(d_in), _lib.ptr(x), nb, s)

    def _bd_pair_ok(self, L, su, sp, x_is_zero):
        _, pu, degu = self.slot[su]
        _, pp, degp = self.slot[sp]
        return not (not BLOCKDIAG_SMOOTH or not L.bd_ok or degu or degp or
                    (pu.degree != pp.degree and not x_is_zero))

    def _lean_pair(self, L, su, sp):
        """The block-diagonal x = 0 start of (su, sp) stores d only (see LEAN_START)."""
        return (LEAN_START and self._bd_pair_ok(L, su, sp, True) and
                min(self.slot[su][1].degree, self.slot[sp][1].degree) >= 2)

    def _cheb_pair(self, L, su, sp, x_is_zero, pre=True, init_done=False):
        """Chebyshev on both diagonal blocks (independent, mgsolve.py:200-206) with
        one block-diagonal kernel per step while both recurrences run.
        init_done: the x = 0 start (r, d, x) was already written by the fused
        restriction (pffmg_restrict_init_bd)."""
        ou, pu, degu = self.slot[su]
        op_, pp, degp = self.slot[sp]
        if not self._bd_pair_ok(L, su, sp, x_is_zero):
            self._cheb(L, 0, su, x_is_zero, pre)
            self._cheb(L, 1, sp, x_is_zero, pre)
            return
        op, coef, s = L.op, self.coef, _lib.stream()
        x, r, rhs, inv, d_in, d_out = L.x, L.cr, L.r, L.inv, L.d0, L.d1
        tu, tp = coef[ou:ou + 1], coef[op_:op_ + 1]
        lean = x_is_zero and self._lean_pair(L, su, sp)
        if x_is_zero and init_done:
            pending = False
        elif x_is_zero:
            _lib.call("pffmg_cheb_init_zero_bd", _lib.ptr(rhs), _lib.ptr(inv), _lib.ptr(tu), _lib.ptr(tp),
                      L.dim * L.V, None if lean else _lib.ptr(r), _lib.ptr(d_in),
                      None if lean else _lib.ptr(x), L.n, s)
            pending = False
        else:
            self._stencil(L, x, L.dim + 1, lambda: op.cheb_init_bd(x, rhs, r, d_in, inv, tu, tp, pre=pre))
            pending = True
        common = min(pu.degree, pp.degree) - 1
        for i in range(common):
            cu, cp = coef[ou + 1 + 2 * i: ou + 3 + 2 * i], coef[op_ + 1 + 2 * i: op_ + 3 + 2 * i]
            if lean and i == 0:
                self._stencil(L, d_in, L.dim + 1,
                              lambda: op.cheb_first_bd(d_in, rhs, d_out, r, x, inv, cu, cp, pre=pre))
            else:
                self._stencil(L, d_in, L.dim + 1,
                              lambda: op.cheb_step_bd(d_in, d_out, r, x, inv, cu, cp, pending, pre=pre))
            pending = False
            d_in, d_out = d_out, d_in
        if pending:                                        # degree 1 from a non-zero x
            _lib.call("pffmg_axpy", 1.0, _lib.ptr(d_in), _lib.ptr(x), L.n, s)
        for k, (o, prm) in enumerate(((ou, pu), (op_, pp))):   # the longer recurrence goes on alone
            b = L.blk(k)
            di, do = d_in[b], d_out[b]
            for i in range(common, prm.degree - 1):
                c = coef[o + 1 + 2 * i: o + 3 + 2 * i]
                self._stencil(L, di, L.dim if k == 0 else 1,
                              lambda: op.cheb_step_dc(k, di, do, r[b], x[b], inv[b], c, False, pre=pre))
                di, do = do, di

    def _smooth(self, l, x_is_zero, init_done=False):
        self._cheb_pair(self.levels[l], ("s", l, 0), ("s", l, 1), x_is_zero, init_done=init_done)

    def _fused_descent_ok(self, l):
        """Restriction into level l can carry level l's smoother start (x = 0)."""
        Lc = self.levels[l]
        return (FUSED_DESCENT and self.comm is None and l >= 1 and
                self._bd_pair_ok(Lc, ("s", l, 0), ("s", l, 1), True))

    def _coarse_into_x(self, pre=True):
        L = self.levels[0]
        ou, pu, degu = self.slot[("c", 0, 0)]
        op_, pp, degp = self.slot[("c", 0, 1)]
        if COARSE_KERNEL and L.coarse_ok and not (degu or degp):
            # the whole coarse_solve in one launch (libpffmg pffmg_coarse_cheb)
            c = self.coef
            _lib.call("pffmg_coarse_cheb", L.op.lat.ref, L.op._sp(pre), _lib.ptr(L.r), _lib.ptr(L.x),
                      _lib.ptr(L.cr), _lib.ptr(L.d0), _lib.ptr(L.inv), _lib.ptr(c[ou:]), pu.degree,
                      _lib.ptr(c[op_:]), pp.degree, _lib.stream())
            return
        self._cheb_pair(L, ("c", 0, 0), ("c", 0, 1), True, pre)

    def _cycle(self, l, init_done=False):                  # mgsolve.py:221-235
        if l == 0:
            self._coarse_into_x()
            return
        L, Lc = self.levels[l], self.levels[l - 1]
        self._smooth(l, True, init_done)
        self._stencil(L, L.x, L.dim + 1, lambda: L.op.residual_dev(_lib.FULL, L.x, L.r, L.res, pre=True))
        if self._fused_descent_ok(l - 1):
            ou, _, _ = self.slot[("s", l - 1, 0)]
            op_, _, _ = self.slot[("s", l - 1, 1)]
            lean = self._lean_pair(Lc, ("s", l - 1, 0), ("s", l - 1, 1))
            self.disc.restrict_init_bd_dev(L.res, Lc.r, l - 1, Lc.flags, Lc.inv, self.coef[ou:ou + 1],
                                           self.coef[op_:op_ + 1], None if lean else Lc.cr, Lc.d0,
                                           None if lean else Lc.x)
            self._cycle(l - 1, init_done=True)
        else:
            self._restrict(l - 1, L.res, Lc.r, L.dim + 1, 0, Lc.flags)
            self._cycle(l - 1)
        self._prolongate(l - 1, Lc.x, L.x, L.dim + 1, 0, L.flags)
        self._smooth(l, False)

    def _block_cycle(self, k, l):                          # mgsolve.py:238-259
        L = self.levels[l]
        if l == 0:
            self._cheb(L, k, ("c", 0, k), True)
            return
        Lc = self.levels[l - 1]
        b = L.blk(k)
        self._cheb(L, k, ("s", l, k), True)
        ncomp = L.dim if k == 0 else 1
        comp0 = 0 if k == 0 else L.dim
        self._stencil(L, L.x[b], ncomp, lambda: L.op.residual_dev(k, L.x[b], L.r[b], L.res[b], pre=True))
        self._restrict(l - 1, L.res[b], Lc.r[Lc.blk(k)], ncomp, comp0, Lc.flags)
        self._block_cycle(k, l - 1)
        self._prolongate(l - 1, Lc.x[Lc.blk(k)], L.x[b], ncomp, comp0, L.flags)
        self._cheb(L, k, ("s", l, k), False)

    def _entry_fused(self, kind):
        """The V-cycle input's masking carries the fine level's smoother start."""
        top = len(self.levels) - 1
        return (kind == "full" and FUSED_DESCENT and self.comm is None and top >= 1 and
                self._bd_pair_ok(self.levels[top], ("s", top, 0), ("s", top, 1), True))

    def _body(self, kind):
        if kind == "full":
            self._cycle(len(self.levels) - 1, init_done=self._entry_fused(kind))
        else:
            for k in range(2):
                self._block_cycle(k, len(self.levels) - 1)

    def run(self, kind, r, out):
        top = self.levels[-1]
        fused = self._entry_fused(kind)

        def entry():
            # r[constrained] = 0 straight from the caller's vector into the fine level's
            # rhs (mgsolve.py:271-272); the recorded cycle then reads fixed buffers only
            if fused:                        # ... together with the smoother's x = 0 start
                t = len(self.levels) - 1
                ou, _, _ = self.slot[("s", t, 0)]
                op_, _, _ = self.slot[("s", t, 1)]
                lean = self._lean_pair(top, ("s", t, 0), ("s", t, 1))
                _lib.call("pffmg_masked_copy_init_bd", _lib.ptr(top.flags), top.V, top.dim + 1, _lib.ptr(r),
                          _lib.ptr(top.r), _lib.ptr(top.inv), _lib.ptr(self.coef[ou:ou + 1]),
                          _lib.ptr(self.coef[op_:op_ + 1]), None if lean else _lib.ptr(top.cr),
                          _lib.ptr(top.d0), None if lean else _lib.ptr(top.x), _lib.stream())
            else:
                _lib.call("pffmg_masked_copy", _lib.ptr(top.flags), top.V, 0, top.dim + 1,
                          _lib.ptr(r), _lib.ptr(top.r), _lib.stream())

        if self.use_graph:
            g = self.graphs.get(kind)
            if g is None:
                entry()
                self._body(kind)                       # warm-up (allocator, lazy attributes)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._body(kind)
                self.graphs[kind] = g
            entry()                                    # (the fused entry state is consumed by a cycle)
            g.replay()
        else:
            entry()
            self._body(kind)
        out.copy_(top.x)

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
        self._args = (degree, coarse_target, coarse_cap)
        self.cycle = _NativeCycle.get(contexts, *self._args)

    def _cycle(self):
        # re-resolved per call: a later build_level_contexts may have detached
        # these contexts from the reusable session (see _Session)
        return _NativeCycle.get(self.contexts, *self._args)

    def __call__(self, r):
        rd = dev(r)
        out = empty(rd.numel())
        self._cycle().run(self.kind, rd, out)
        return like(out, r)

    def _pffmg_into(self, src, dst):
        self._cycle().run(self.kind, src, dst)

"""Drop-in twin of the reference operator layer (model.py) on sm_100a kernels.

`PhaseFieldOperator(space, state, mask, params, split, threads=1)` has the
constructor and protocol of reference model.py:242-413 (apply, apply_block,
diagonal, blocks, mask, state, params, space, n_dofs).  Construction uploads
the linearisation point U, phi_tilde and the packed constraint bits; every
application is ONE fused kernel launch (libpffmg `pffmg_apply`) that gathers
the cell's vertex data, interpolates to the 2-point Gauss points, evaluates
the degraded stress / phase-field coupling / reaction, integrates and sums
the vertex contributions deterministically.  The per-QP coefficient tables
the reference caches in `_build_caches` (model.py:270-309) are recomputed on
the fly instead of being streamed from HBM (fewer bytes per vmult).

Vectors may be numpy arrays (copied to the GPU and back) or CUDA tensors
(zero copy); the result has the kind of the input.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from enum import Enum
from typing import Callable, Optional

import contextlib
import os

import numpy as np
import torch

from . import _lib
from .arrays import dev, empty, host, is_tensor, like, pack_flags, unpack_flags
from .lattice import LatticeMesh, device_lattice

__all__ = ["SplitKind", "MaterialParams", "LinearizationState", "ConstraintMask", "residual",
           "PhaseFieldOperator", "extrapolate", "degradation", "jacobian_vmult", "diagonal",
           "crack_energy", "bulk_energy", "fracture_volume", "boundary_load"]


class SplitKind(Enum):
    NOSPLIT = "none"
    MIEHE = "miehe"


@dataclass
class MaterialParams:
    """Same fields as reference model.py:89-103."""
    mu: float
    lam: float
    g_c: float
    kappa: float = 1e-10
    eps: float = 1.0
    pressure_fn: Optional[Callable[[float], float]] = None
    modulus_field: Optional[Callable[[np.ndarray], np.ndarray]] = None
    split_band: float = 0.0

    def pressure(self, t):
        return float(self.pressure_fn(t)) if self.pressure_fn is not None else 0.0


@dataclass
class LinearizationState:
    """Same fields as reference model.py:106-119 (arrays may live on the GPU)."""
    U: object
    U_prev1: object
    U_prev2: object
    t: float
    t_prev1: float
    t_prev2: float
    phi_tilde: object

    def with_U(self, U):
        return replace(self, U=U)


@dataclass
class ConstraintMask:
    """Same fields and semantics as reference fem.py:129-145."""
    is_constrained: np.ndarray
    inhomogeneity: np.ndarray

    @classmethod
    def empty(cls, n_dofs):
        return cls(np.zeros(n_dofs, dtype=bool), np.zeros(n_dofs))

    def combined_with(self, flags, values):
        is_c = self.is_constrained | flags
        vals = np.where(self.is_constrained, self.inhomogeneity, np.where(flags, values, 0.0))
        return ConstraintMask(is_c, vals)


class DeviceMask:
    """A constraint mask that lives on the GPU as packed per-vertex bits; the
    numpy view (`is_constrained`) is materialised lazily on first access."""

    def __init__(self, flags, n_comp, V, inhomogeneity=None):
        self.flags = flags
        self.n_comp = n_comp
        self.V = V
        self._host = None
        self._host_fn = None          # optional lazy host view (e.g. the caller's own arrays)
        self._inh = inhomogeneity     # array, callable (lazy) or None (zeros)

    @property
    def is_constrained(self):
        if self._host is None:
            self._host = (self._host_fn() if self._host_fn is not None
                          else host(unpack_flags(self.flags, self.n_comp, self.V)))
        return self._host

    @property
    def inhomogeneity(self):
        if self._inh is None:
            self._inh = np.zeros(self.n_comp * self.V)
        elif callable(self._inh):
            self._inh = self._inh()
        return self._inh


def extrapolate(phi_prev1, phi_prev2, t, t_prev1, t_prev2):
    """Reference model.py:122-132 (host helper, not on the hot path)."""
    phi_prev1 = np.asarray(phi_prev1, dtype=float)
    dt = t_prev1 - t_prev2
    if dt <= 0.0:
        return np.clip(phi_prev1, 0.0, 1.0)
    return np.clip(phi_prev1 + (t - t_prev1) * (phi_prev1 - np.asarray(phi_prev2, float)) / dt, 0.0, 1.0)


def degradation(phi, kappa):
    """Reference model.py:135-137."""
    return (1.0 - kappa) * np.square(phi) + kappa


def _split_code(split):
    v = getattr(split, "value", split)
    if v in ("none", 0, None):
        return 0
    if v in ("miehe", 1):
        return 1
    raise ValueError(f"unknown split kind {split!r}")


class PhaseFieldOperator:
    """Matrix-free constrained Jacobian of one level (reference model.py:242-413)."""

    def __init__(self, space, state, mask, params, split, threads=1, *, _flags=None, _rho=None, _ptab=None,
                 _no_table=False):
        _lib.require_cuda()
        self.space = space
        self.state = state
        self.mask = mask
        self.params = params
        self.split = split
        self.threads = max(1, int(threads))
        self.lat = device_lattice(space.mesh)
        self.dim = self.lat.dim
        self.nc = self.dim + 1
        V = self.lat.n_vertices
        self.V = V
        code = _split_code(split)
        self._U = dev(state.U)
        self._pt = dev(state.phi_tilde)
        if _flags is None and not _no_table:
            # the reference caches every coefficient at construction
            # (model.py:260, 270-309): a caller's CUDA state is snapshotted so a
            # later in-place update of state.U cannot mix old and new
            # coefficients (internal callers own their buffers and pass _flags;
            # the one-shot helpers below use the operator immediately)
            if is_tensor(state.U) and self._U.data_ptr() == state.U.data_ptr():
                self._U = self._U.clone()
            if is_tensor(state.phi_tilde) and self._pt.data_ptr() == state.phi_tilde.data_ptr():
                self._pt = self._pt.clone()
        if self._U.numel() != self.nc * V or self._pt.numel() != V:
            raise ValueError(f"state sizes {self._U.numel()}/{self._pt.numel()} do not match "
                             f"the level ({self.nc}x{V} dofs)")
        self._flags = _flags if _flags is not None else pack_flags(mask.is_constrained, self.nc, V)
        if _rho is not None:
            self._rho = _rho
        else:
            self._rho = self._modulus_table() if params.modulus_field is not None else None
        st = _lib.State()
        st.mu, st.lam, st.g_c = float(params.mu), float(params.lam), float(params.g_c)
        st.kappa, st.eps = float(params.kappa), float(params.eps)
        st.pressure = float(params.pressure(state.t))
        st.split = code
        st.split_band = float(getattr(params, "split_band", 0.0) or 0.0)
        st.U = self._U.data_ptr()
        st.phi_tilde = self._pt.data_ptr()
        st.rho = self._rho.data_ptr() if self._rho is not None else None
        st.flags = self._flags.data_ptr()
        self._st = st
        import ctypes
        self._stp = ctypes.byref(st)
        # same state with PFFMG_HINT_PREMASKED: for internal callers whose input
        # vectors are zero at constrained dofs by construction (V-cycle, CG)
        st_pre = _lib.State()
        ctypes.pointer(st_pre)[0] = st
        st_pre.hints = 1
        self._st_pre = st_pre
        self._stp_pre = ctypes.byref(st_pre)
        # ... and with PFFMG_HINT_ENDS: only the first and last owned plane (slab boundaries)
        st_ends = _lib.State()
        ctypes.pointer(st_ends)[0] = st
        st_ends.hints = 2
        self._st_ends = st_ends
        self._stp_ends = ctypes.byref(st_ends)
        st_pre_ends = _lib.State()
        ctypes.pointer(st_pre_ends)[0] = st
        st_pre_ends.hints = 3
        self._st_pre_ends = st_pre_ends
        self._stp_pre_ends = ctypes.byref(st_pre_ends)
        self._scope = None          # row scope of the slab-overlapped stencils (see scope())
        # per-QP a_phiphi of the phi block, cached like _build_caches does
        # (model.py:260, 304-308): NoSplit Q2 and isotropic Q1 levels (phi
        # block, block-diagonal smoother)
        self._ptab = None
        info = self.lat.info
        h = np.asarray(info.h, float)
        order = getattr(info, "order", 1)
        if (code == 0 and (order == 2 or np.all(h == h[0])) and not _no_table
                and os.environ.get("PFFMG_PHI_TABLE", "1") != "0"):
            if _ptab is not None:            # a table already built from this state (mgsolve._Session)
                self._ptab = _ptab
                for st in (self._st, self._st_pre, self._st_ends, self._st_pre_ends):
                    st.phi_coef = _ptab.data_ptr()
            else:
                self._ptab = empty((9 if order == 2 else 1 << self.dim) * self.lat.n_lattice_cells)
                self.build_phi_coef()

    def build_phi_coef(self):
        """(Re)build the phi-block coefficient table from the current U (device
        work on the current stream; graph-capturable) and point the states at it."""
        if self._ptab is None:
            return
        for st in (self._st, self._st_pre, self._st_ends, self._st_pre_ends):
            st.phi_coef = None
        _lib.call("pffmg_phi_coef", self.lat.ref, self._stp, _lib.ptr(self._ptab), _lib.stream())
        for st in (self._st, self._st_pre, self._st_ends, self._st_pre_ends):
            st.phi_coef = self._ptab.data_ptr()

    def _rebind(self, U, phi_tilde, flags):
        """Point the operator at other device buffers of the same sizes (used
        to detach an earlier generation of solver contexts, mgsolve._Session)."""
        self._U, self._pt, self._flags = U, phi_tilde, flags
        if self._ptab is not None:
            self._ptab = self._ptab.clone()
        for st in (self._st, self._st_pre, self._st_ends, self._st_pre_ends):
            st.U = U.data_ptr()
            st.phi_tilde = phi_tilde.data_ptr()
            st.flags = flags.data_ptr()
            if self._ptab is not None:
                st.phi_coef = self._ptab.data_ptr()
        if isinstance(self.mask, DeviceMask):
            self.mask.flags = flags

    # -- reference surface --------------------------------------------------
    @property
    def n_dofs(self):
        return self.nc * self.V

    @property
    def blocks(self):
        return (slice(0, self.dim * self.V), slice(self.dim * self.V, self.nc * self.V))

    @property
    def flags(self):
        """Packed constraint bits on the device."""
        return self._flags

    def apply(self, v, out=None):
        """G~ v with constrained rows = identity (model.py:368-375).  `out`
        (optional, not in the reference signature) receives the result.
        Pinned host tensors take the pipelined host path (pffmg_apply_host)."""
        if _pinned_f64(v) and (out is None or _pinned_f64(out)) and self.lat.info.own == (0, 0):
            return self._apply_host(v, out)
        if (PAGEABLE_PIPELINE and _plain_f64(v) and (out is None or _plain_f64(out, True))
                and v.size == self.n_dofs >= PAGEABLE_MIN and self.lat.info.own == (0, 0)):
            return self._apply_pageable(v, out)
        x = dev(v)
        if x.numel() != self.n_dofs:
            raise ValueError(f"expected {self.n_dofs} dofs, got {x.numel()}")
        y = out if (is_tensor(out) and out.is_cuda) else empty(self.n_dofs)
        self.apply_dev(_lib.FULL, x, y)
        if y is out:
            return out
        return like(y, v, out)

    def _apply_host(self, v, out):
        n = self.n_dofs
        if v.numel() != n or (out is not None and out.numel() != n):
            raise ValueError(f"expected {n} dofs, got {v.numel()}")
        if out is None:
            out = torch.empty(n, dtype=torch.float64, pin_memory=True)
        bufs = getattr(self, "_host_bufs", None)
        if bufs is None:
            bufs = self._host_bufs = (empty(n), empty(n))
        po = self.lat.plane_off_host
        strips = int(max(1, min(8, round(8 * n / (4 << 20)))))  # ~4 MiB per strip and direction
        _lib.call("pffmg_apply_host", self.lat.ref, self._stp, _lib.FULL, C_ptr(v), C_ptr(out),
                  _lib.ptr(bufs[0]), _lib.ptr(bufs[1]), None if po is None else po.ctypes.data,
                  strips, _lib.stream())
        torch.cuda.current_stream().synchronize()
        return out

    def _apply_pageable(self, v, out):
        """numpy in / numpy out (what the reference's drivers pass): threaded
        staging through the library's page-locked buffers, pipelined with the
        link copies and the stencil (pffmg_apply_pageable)."""
        n = self.n_dofs
        if out is None:
            out = np.empty(n, dtype=np.float64)
        elif out.size != n:
            raise ValueError(f"expected {n} dofs, got {out.size}")
        bufs = getattr(self, "_host_bufs", None)
        if bufs is None:
            bufs = self._host_bufs = (empty(n), empty(n))
        po = self.lat.plane_off_host
        strips = int(max(1, min(8, round(8 * n / (4 << 20)))))
        _lib.call("pffmg_apply_pageable", self.lat.ref, self._stp, _lib.FULL, v.ctypes.data, out.ctypes.data,
                  _lib.ptr(bufs[0]), _lib.ptr(bufs[1]), None if po is None else po.ctypes.data,
                  strips, _lib.stream())
        return out

    def apply_block(self, which, v_block):
        """Diagonal block action, 0 = displacement, 1 = phase field (model.py:377-392)."""
        x = dev(v_block)
        n = self.dim * self.V if which == 0 else self.V
        if x.numel() != n:
            raise ValueError(f"block {which} expects {n} entries, got {x.numel()}")
        out = empty(n)
        self.apply_dev(which, x, out)
        return like(out, v_block)

    def diagonal(self):
        """Exact diagonal, constrained entries 1.0 (model.py:394-413), as numpy
        like the reference; `diagonal_dev` fills a CUDA tensor instead."""
        out = empty(self.n_dofs)
        self.diagonal_dev(out)
        return host(out)

    # -- device-level entry points (no conversions) --------------------------
    def _sp(self, pre):
        if self._scope == "ends":
            return self._stp_pre_ends if pre else self._stp_ends
        return self._stp_pre if pre else self._stp

    def _lref(self):
        sc = self._scope
        return self.lat.ref if sc is None or sc == "ends" else self.lat.rows(sc[1], sc[2])

    @contextlib.contextmanager
    def scope(self, sc):
        """Restrict the *_dev stencil calls to some vertex planes of a slab:
        ("rows", lo, hi) finalises planes [lo, hi) only, "ends" the first and
        the last owned plane (PFFMG_HINT_ENDS) -- the interior / boundary
        halves of a halo-overlapped stencil (dist_solver.DistGMG)."""
        old, self._scope = self._scope, sc
        try:
            yield self
        finally:
            self._scope = old

    def apply_dev(self, which, x, out, pre=False):
        _lib.call("pffmg_apply", self._lref(), self._sp(pre), which, _lib.ptr(x), _lib.ptr(out),
                  _lib.stream())

    def apply_rows_dev(self, which, x, out, lo, hi, pre=False):
        """apply_dev finalising only vertex planes [lo, hi) of the last axis."""
        _lib.call("pffmg_apply", self.lat.rows(lo, hi), self._sp(pre), which, _lib.ptr(x), _lib.ptr(out),
                  _lib.stream())

    def apply_ends_dev(self, which, x, out):
        """apply_dev finalising only the first and the last owned plane (one launch)."""
        _lib.call("pffmg_apply", self.lat.ref, self._stp_ends, which, _lib.ptr(x), _lib.ptr(out),
                  _lib.stream())

    def residual_dev(self, which, x, b, out, pre=False):
        _lib.call("pffmg_residual", self._lref(), self._sp(pre), which, _lib.ptr(x), _lib.ptr(b),
                  _lib.ptr(out), _lib.stream())

    def semilinear_dev(self, out):
        """out = A(U) of the linearisation state, constrained rows zeroed (model.py:420-460)."""
        _lib.call("pffmg_semilinear_residual", self.lat.ref, self._stp, _lib.ptr(out), _lib.stream())

    def diagonal_dev(self, out):
        _lib.call("pffmg_diagonal", self.lat.ref, self._stp, _lib.ptr(out), _lib.stream())

    def cheb_step_dev(self, which, d_in, d_out, r, x, inv, c_dd, c_dr, x_add_din=False, pre=False):
        _lib.call("pffmg_cheb_step", self._lref(), self._sp(pre), which, _lib.ptr(d_in),
                  _lib.ptr(d_out), _lib.ptr(r), _lib.ptr(x), _lib.ptr(inv), c_dd, c_dr,
                  int(x_add_din), _lib.stream())

    def cheb_init_dev(self, which, x, b, r, d, inv, theta, pre=False):
        _lib.call("pffmg_cheb_init", self._lref(), self._sp(pre), which, _lib.ptr(x), _lib.ptr(b),
                  _lib.ptr(r), _lib.ptr(d), _lib.ptr(inv), theta, _lib.stream())

    # device-coefficient forms: scalars read from `coef` (a CUDA tensor view) at run time
    def cheb_step_dc(self, which, d_in, d_out, r, x, inv, coef, x_add_din=False, pre=False):
        _lib.call("pffmg_cheb_step_dc", self._lref(), self._sp(pre), which, _lib.ptr(d_in),
                  _lib.ptr(d_out), _lib.ptr(r), _lib.ptr(x), _lib.ptr(inv), _lib.ptr(coef),
                  int(x_add_din), _lib.stream())

    def cheb_step_bd(self, d_in, d_out, r, x, inv, coef_u, coef_p, x_add_din=False, pre=False):
        """Both diagonal blocks' Chebyshev steps in one kernel (full-length vectors)."""
        _lib.call("pffmg_cheb_step_bd", self._lref(), self._sp(pre), _lib.ptr(d_in), _lib.ptr(d_out),
                  _lib.ptr(r), _lib.ptr(x), _lib.ptr(inv), _lib.ptr(coef_u), _lib.ptr(coef_p),
                  int(x_add_din), _lib.stream())

    def cheb_first_bd(self, d_in, rhs, d_out, r, x, inv, coef_u, coef_p, pre=False):
        """First step after the lean x = 0 start (r = rhs, x = d_in not stored): both blocks."""
        _lib.call("pffmg_cheb_first_bd", self._lref(), self._sp(pre), _lib.ptr(d_in), _lib.ptr(rhs),
                  _lib.ptr(d_out), _lib.ptr(r), _lib.ptr(x), _lib.ptr(inv), _lib.ptr(coef_u), _lib.ptr(coef_p),
                  _lib.stream())

    def cheb_first_dc(self, which, d_in, rhs, d_out, r, x, inv, coef, pre=False):
        """First step after the lean x = 0 start of one block."""
        _lib.call("pffmg_cheb_first_dc", self._lref(), self._sp(pre), which, _lib.ptr(d_in), _lib.ptr(rhs),
                  _lib.ptr(d_out), _lib.ptr(r), _lib.ptr(x), _lib.ptr(inv), _lib.ptr(coef), _lib.stream())

    def cheb_init_bd(self, x, b, r, d, inv, theta_u, theta_p, pre=False):
        _lib.call("pffmg_cheb_init_bd", self._lref(), self._sp(pre), _lib.ptr(x), _lib.ptr(b), _lib.ptr(r),
                  _lib.ptr(d), _lib.ptr(inv), _lib.ptr(theta_u), _lib.ptr(theta_p), _lib.stream())

    def cheb_init_dc(self, which, x, b, r, d, inv, theta, pre=False):
        _lib.call("pffmg_cheb_init_dc", self._lref(), self._sp(pre), which, _lib.ptr(x), _lib.ptr(b),
                  _lib.ptr(r), _lib.ptr(d), _lib.ptr(inv), _lib.ptr(theta), _lib.stream())

    # -- helpers ---------------------------------------------------------------
    def _modulus_table(self):
        return _modulus_table(self.space, self.lat, self.params)


def _modulus_table(space, lat, params):
    """rho(x_q) per lattice cell and QP (model.py:284-287)."""
    info = lat.info
    Q = 9 if getattr(info, "order", 1) == 2 else 2 ** lat.dim
    ncell_lat = int(np.prod(info.ncell))
    table = np.ones((ncell_lat, Q))
    coords = getattr(space, "qp_coords", None)
    if coords is not None and info.cell_perm is not None:
        rho = np.asarray(params.modulus_field(coords), dtype=float)
        table[info.cell_perm] = rho
    else:
        coords = _lattice_qp_coords(space.mesh)
        table = np.asarray(params.modulus_field(coords), dtype=float).reshape(ncell_lat, Q)
    return dev(table.ravel())


# numpy vectors of at least PAGEABLE_MIN dofs go through pffmg_apply_pageable
# (PFFMG_PAGEABLE_PIPELINE=0: plain pageable copies around the device apply)
PAGEABLE_PIPELINE = os.environ.get("PFFMG_PAGEABLE_PIPELINE", "1") != "0"
PAGEABLE_MIN = 1 << 20


def _plain_f64(a, writeable=False):
    return (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.ndim == 1
            and a.flags.c_contiguous and a.flags.aligned and (a.flags.writeable or not writeable))


def _pinned_f64(t):
    return (is_tensor(t) and not t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
            and t.is_pinned())


def C_ptr(t):
    import ctypes
    return ctypes.c_void_p(t.data_ptr())


def _lattice_qp_coords(mesh):
    """QP coordinates of every lattice cell (lattice order), fem.py:181-182."""
    if getattr(mesh, "order", 1) == 2:                    # Q2: 3x3 Gauss, qx + 3 qy
        g = np.array([0.5 - 0.5 * np.sqrt(0.6), 0.5, 0.5 + 0.5 * np.sqrt(0.6)])
        pts = np.stack([np.tile(g, 3), np.repeat(g, 3)], axis=1)
        nx, ny = (int(v) for v in mesh.ncell)
        cy, cx = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        lo = mesh.lo[None, :] + np.stack([cx.ravel(), cy.ravel()], axis=1) * mesh.cell_size
        return lo[:, None, :] + pts[None, :, :] * mesh.cell_size
    dim = mesh.dim
    g = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])
    idx = np.arange(2 ** dim)
    pts = np.stack([g[(idx >> a) & 1] for a in range(dim)], axis=1)
    grids = np.meshgrid(*[np.arange(e) for e in mesh.ncell[::-1]], indexing="ij")
    base = np.stack([gr.ravel() for gr in grids[::-1]], axis=1) + mesh.kmin
    lo = base.astype(float) * mesh.cell_size
    return lo[:, None, :] + pts[None, :, :] * mesh.cell_size


def residual(space, state, mask, params, split, threads=1):
    """Discrete semilinear form A_h(U) with constrained rows zeroed (reference
    model.py:420-460), on the GPU.  Returns the kind of `state.U`."""
    # one-shot operators: the full operator / residual / diagonal never read
    # the phi-block table, so none is built
    op = PhaseFieldOperator(space, state, mask, params, split, threads, _no_table=True)
    out = empty(op.n_dofs)
    op.semilinear_dev(out)
    return like(out, state.U)


def jacobian_vmult(space, state, mask, params, split, v, threads=1):
    return PhaseFieldOperator(space, state, mask, params, split, threads, _no_table=True).apply(v)


def diagonal(space, state, mask, params, split, threads=1):
    return PhaseFieldOperator(space, state, mask, params, split, threads, _no_table=True).diagonal()


# ------------------------------------------------------------------ QoIs

def _qoi(space, U, params, split, t, kind):
    """One deterministic device reduction (libpffmg pffmg_qoi) -> float."""
    import ctypes
    _lib.require_cuda()
    lat = device_lattice(space.mesh)
    Ud = dev(U)
    if Ud.numel() != (lat.dim + 1) * lat.n_vertices:
        raise ValueError(f"U has {Ud.numel()} entries, expected {(lat.dim + 1) * lat.n_vertices}")
    st = _lib.State()
    st.mu, st.lam, st.g_c = float(params.mu), float(params.lam), float(params.g_c)
    st.kappa, st.eps = float(params.kappa), float(params.eps)
    st.pressure = float(params.pressure(t)) if t is not None else 0.0
    st.split = _split_code(split)
    st.split_band = float(getattr(params, "split_band", 0.0) or 0.0)
    st.U = Ud.data_ptr()
    rho = None
    if kind == 1 and getattr(params, "modulus_field", None) is not None:
        rho = _modulus_table(space, lat, params)
        st.rho = rho.data_ptr()
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    _lib.call("pffmg_qoi", lat.ref, ctypes.byref(st), int(kind), _lib.ptr(out), _lib.stream())
    return float(out.item())


def crack_energy(space, state, params):
    """Regularised surface energy (reference model.py:472-480)."""
    return _qoi(space, state.U, params, SplitKind.NOSPLIT, None, 0)


def bulk_energy(space, state, params, split):
    """Degraded tensile + compressive elastic energy + pressure work (model.py:483-497)."""
    return _qoi(space, state.U, params, split, state.t, 1)


def fracture_volume(space, U):
    """Integral of (1 - phi) (model.py:500-504)."""
    p = MaterialParams(mu=0.0, lam=0.0, g_c=0.0, eps=1.0)
    return _qoi(space, U, p, SplitKind.NOSPLIT, None, 2)


BOUNDARY_IDS = (0, 1, 2, 3)     # mesh.BoundaryId: OUTER, FIXED, LOADED, TRACTION_FREE (mesh.py:24-28)


def _face_points(dim, axis, side):
    """Reference-cell face quadrature points (fem.py:265-281 order)."""
    g = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])
    other = [a for a in range(dim) if a != axis]
    if dim == 2:
        ref = np.zeros((2, dim))
        ref[:, other[0]] = g
    else:
        g0, g1 = np.meshgrid(g, g, indexing="ij")
        ref = np.zeros((4, dim))
        ref[:, other[0]] = g0.ravel()
        ref[:, other[1]] = g1.ravel()
    ref[:, axis] = float(side)
    return ref


def boundary_load(space, state, params, split, boundary, direction):
    """Traction component `direction` integrated over the faces tagged
    `boundary` (reference model.py:511-547): g(phi) rho sigma+ + rho sigma-
    at the face Gauss points, one deterministic device reduction
    (libpffmg pffmg_boundary_load)."""
    import ctypes
    if int(boundary) not in BOUNDARY_IDS:
        raise ValueError(f"unknown boundary tag {boundary!r}")
    _lib.require_cuda()
    mesh = space.mesh
    lat = device_lattice(mesh)
    if getattr(lat.info, "order", 1) != 1:
        raise ValueError("boundary_load is defined for the reference's Q1 elements only")
    dim = lat.dim
    if not 0 <= int(direction) < dim:
        raise ValueError(f"direction {direction!r} out of range for dim {dim}")
    rows = np.nonzero(np.asarray(mesh.bf_tag) == int(boundary))[0]
    cells = np.asarray(mesh.bf_cell)[rows]
    faces = np.asarray(mesh.bf_face)[rows]
    if isinstance(mesh, LatticeMesh):
        lcell = mesh.lattice_cell_index(cells)
    else:
        lcell = np.asarray(lat.info.cell_perm, dtype=np.int64)[cells]
    Ud = dev(state.U)
    if Ud.numel() != (dim + 1) * lat.n_vertices:
        raise ValueError(f"U has {Ud.numel()} entries, expected {(dim + 1) * lat.n_vertices}")
    rho = None
    if getattr(params, "modulus_field", None) is not None and len(rows):
        if isinstance(mesh, LatticeMesh):
            lo = mesh.cell_lower_corners(cells)
        else:
            lo = np.asarray(mesh.vertices)[np.asarray(mesh.cells)[cells, 0]]
        h = np.asarray(mesh.cell_size, dtype=float)
        coords = np.empty((len(rows), 2 ** (dim - 1), dim))
        for f in np.unique(faces):
            sel = faces == f
            coords[sel] = lo[sel][:, None, :] + _face_points(dim, int(f) // 2, int(f) % 2)[None, :, :] * h
        rho = dev(np.asarray(params.modulus_field(coords), dtype=float).ravel())
    st = _lib.State()
    st.mu, st.lam, st.g_c = float(params.mu), float(params.lam), float(params.g_c)
    st.kappa, st.eps = float(params.kappa), float(params.eps)
    st.split = _split_code(split)
    st.split_band = float(getattr(params, "split_band", 0.0) or 0.0)
    st.U = Ud.data_ptr()
    fc = dev(lcell.astype(np.int64), torch.int64)
    ff = dev(faces.astype(np.int32), torch.int32)
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    _lib.call("pffmg_boundary_load", lat.ref, ctypes.byref(st), _lib.ptr(fc), _lib.ptr(ff), len(rows),
              int(direction), _lib.ptr(rho), _lib.ptr(out), _lib.stream())
    return float(out.item())

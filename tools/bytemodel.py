"""Algorithmic HBM bytes of every libpffmg launch (SURVEY §8d "Solve-level HBM
fraction": sum of kernel algorithmic bytes / T_solve / P).

`Recorder` wraps `_lib.call` and adds, per entry point, the compulsory traffic
of the call from its arguments: every vector the kernel must read or write
once (8 B per fp64 entry), the packed constraint flags (1 B per vertex), and
the linearisation state the operator kernels recompute their coefficients from
(U and phi_tilde, or the per-QP a_phiphi table where the phi block reads it).
Run a Newton step eagerly (PFFMG_GRAPHS=0: the same kernels the graphs replay)
inside `with Recorder() as rec:` and read `rec.total` / `rec.by_name`.

Two operator models are summed side by side:
  * "F" -- what these kernels must move (coefficients recomputed: state in);
  * "C" -- the reference algorithm's cached tables instead of the state
    (SURVEY §8d B_C: 8 Q (2 + d(d+1)/2) C for the full operator, 8 Q C per
    block), the denominator of the vmult roofline.
"""
from __future__ import annotations

import ctypes as C
from collections import defaultdict

from paper_1902_08112_b200 import _lib

F8 = 8


def _lat(a):
    return a._obj if hasattr(a, "_obj") else a


def _geom(lat):
    L = _lat(lat)
    dim = int(L.dim)
    V = int(L.n_vertices)
    if int(L.order) == 2:
        cells, Q = int(L.nx) * int(L.ny), 9
    else:
        cells = int(L.nx) * int(L.ny) * (int(L.nz) if dim == 3 else 1)
        Q = 2 ** dim
    return dim, V, cells, Q


def _state(st):
    return _lat(st)


def _op_parts(lat, st, which):
    """(vector components touched, state bytes model F, table bytes model C)."""
    dim, V, cells, Q = _geom(lat)
    nc = dim + 1
    S = _state(st)
    has_tab = bool(S.phi_coef)
    if which == _lib.FULL:
        comps, f_state = nc, F8 * (nc + 1) * V
        c_tab = F8 * Q * (2 + dim * (dim + 1) // 2) * cells
    elif which == _lib.UBLOCK:
        comps, f_state, c_tab = dim, F8 * V, F8 * Q * cells
    elif which == _lib.PBLOCK:
        comps = 1
        f_state = F8 * Q * cells if has_tab else F8 * (nc + 1) * V
        c_tab = F8 * Q * cells
    else:                                     # BLOCKDIAG: both diagonal blocks
        comps = nc
        f_state = F8 * V + (F8 * Q * cells if has_tab else F8 * (nc + 1) * V)
        c_tab = 2 * F8 * Q * cells
    return comps, V, f_state, c_tab


def _op(lat, st, which, nvec):
    """Operator launch touching `nvec` block vectors (+ state, flags)."""
    comps, V, f_state, c_tab = _op_parts(lat, st, which)
    vec = F8 * comps * V * nvec + V
    return vec + f_state, vec + c_tab


def _vec(n, k):
    b = F8 * int(n) * k
    return b, b


def _transfer(coarse, fine, ncomp, nf_vec, nc_vec, flags_fine=False, flags_coarse=False):
    _, Vc, _, _ = _geom(coarse)
    _, Vf, _, _ = _geom(fine)
    b = F8 * int(ncomp) * (nf_vec * Vf + nc_vec * Vc) + (Vf if flags_fine else 0) + (Vc if flags_coarse else 0)
    return b, b


def _full_n(lat):
    dim, V, _, _ = _geom(lat)
    return (dim + 1) * V


MODEL = {
    "pffmg_apply": lambda a: _op(a[0], a[1], int(a[2]), 2),                 # v in, out
    "pffmg_residual": lambda a: _op(a[0], a[1], int(a[2]), 3),              # x, b in, out
    "pffmg_cheb_step": lambda a: _op(a[0], a[1], int(a[2]), 7),             # d r x D^-1 in; r d x out
    "pffmg_cheb_step_dc": lambda a: _op(a[0], a[1], int(a[2]), 7),
    "pffmg_cheb_init": lambda a: _op(a[0], a[1], int(a[2]), 6),             # x b D^-1 in; r d x out
    "pffmg_cheb_init_dc": lambda a: _op(a[0], a[1], int(a[2]), 6),
    "pffmg_cheb_step_bd": lambda a: _op(a[0], a[1], _lib.BLOCKDIAG, 7),
    "pffmg_cheb_init_bd": lambda a: _op(a[0], a[1], _lib.BLOCKDIAG, 6),
    "pffmg_coarse_cheb": lambda a: _op(a[0], a[1], _lib.BLOCKDIAG, 4),      # b D^-1 in, x out (+ r, d on chip)
    "pffmg_diagonal": lambda a: _op(a[0], a[1], _lib.FULL, 1),
    "pffmg_semilinear_residual": lambda a: _op(a[0], a[1], _lib.FULL, 1),
    "pffmg_phi_coef": lambda a: (lambda g: (F8 * (g[0] + 2) * g[1] + F8 * g[3] * g[2],) * 2)(_geom(a[0])),
    "pffmg_restrict": lambda a: _transfer(a[0], a[1], a[2], 1, 1, flags_coarse=bool(a[6])),
    "pffmg_restrict_init_bd": lambda a: (lambda g: (F8 * (g[0] + 1) * (_geom(a[1])[1] + 4 * g[1]) + g[1],) * 2)(
        _geom(a[0])),                                                       # vf in; vc, D^-1 in; r d x out
    "pffmg_prolongate": lambda a: _transfer(a[0], a[1], a[2], 2 if int(a[7]) else 1, 1, flags_fine=bool(a[6])),
    "pffmg_inject_f64": lambda a: _transfer(a[0], a[1], a[2], 0, 2),
    "pffmg_inject_flags": lambda a: (2 * _geom(a[0])[1],) * 2,
    "pffmg_masked_copy": lambda a: (F8 * 2 * int(a[1]) * int(a[3]) + int(a[1]),) * 2,
    "pffmg_masked_copy_init_bd": lambda a: (F8 * 6 * int(a[1]) * int(a[2]) + int(a[1]),) * 2,
    "pffmg_cheb_init_zero_bd": lambda a: _vec(a[8], 5),
    "pffmg_cheb_init_zero": lambda a: _vec(a[6], 5),
    "pffmg_cheb_init_zero_dc": lambda a: _vec(a[6], 5),
    "pffmg_jacobi_update": lambda a: _vec(a[4], 4),
    "pffmg_jacobi_update_dc": lambda a: _vec(a[4], 4),
    "pffmg_reciprocal": lambda a: _vec(a[2], 2),
    "pffmg_axpy": lambda a: _vec(a[3], 3),
    "pffmg_axpby": lambda a: _vec(a[4], 3),
    "pffmg_scale": lambda a: _vec(a[2], 2),
    "pffmg_copy": lambda a: _vec(a[2], 2),
    "pffmg_sub": lambda a: _vec(a[3], 3),
    "pffmg_dot": lambda a: _vec(a[2], 2),
    "pffmg_dot_scaled": lambda a: _vec(a[3], 3),
    # one MGS step j: V_0..V_j and w read, w written (the one-launch form)
    "pffmg_arnoldi_mgs": lambda a: _vec(a[4], int(a[2]) + 3),
    "pffmg_multi_axpy": lambda a: _vec(a[5], int(a[2]) + 2),
    "pffmg_cg_start": lambda a: _vec(a[5], 5),
    "pffmg_cg_step": lambda a: _vec(a[5], (2, 5, 3)[int(a[7])]),
    "pffmg_active_set": lambda a: (F8 * 4 * int(a[7]) + 2 * int(a[7]),) * 2,
    "pffmg_pack_flags": lambda a: ((int(a[1]) + 1) * int(a[2]),) * 2,
    "pffmg_unpack_flags": lambda a: ((int(a[1]) + 1) * int(a[2]),) * 2,
}


class Recorder:
    """Context manager: counts launches and algorithmic bytes of libpffmg calls."""

    def __init__(self):
        self.launches = 0
        self.total_F = 0
        self.total_C = 0
        self.by_name = defaultdict(lambda: [0, 0, 0])
        self.unmodelled = set()

    def _call(self, name, *args):
        self._orig(name, *args)
        if name in ("pffmg_version", "pffmg_device_sm_count", "pffmg_injection_map", "pffmg_qoi",
                    "pffmg_boundary_load"):
            return
        fn = MODEL.get(name)
        rec = self.by_name[name]
        rec[0] += 1
        self.launches += 1
        if fn is None:
            self.unmodelled.add(name)
            return
        bf, bc = fn(args)
        rec[1] += bf
        rec[2] += bc
        self.total_F += bf
        self.total_C += bc

    def __enter__(self):
        self._orig = _lib.call
        _lib.call = self._call
        return self

    def __exit__(self, *exc):
        _lib.call = self._orig

    def summary(self):
        return {"launches": self.launches, "bytes_F": self.total_F, "bytes_C": self.total_C,
                "unmodelled": sorted(self.unmodelled),
                "by_name": {k: {"launches": v[0], "bytes_F": v[1], "bytes_C": v[2]}
                            for k, v in sorted(self.by_name.items(), key=lambda kv: -kv[1][1])}}

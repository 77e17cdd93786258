"""ctypes binding of libpffmg.so (the C ABI declared in include/pffmg.h).

The shared library is built in-tree (`make -C paper_1902_08112_b200/csrc`,
or `__graft_entry__.build()`).  There is no fallback: if the library or a
CUDA device is missing, the product path raises.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpffmg.so")

FULL, UBLOCK, PBLOCK, BLOCKDIAG = -1, 0, 1, 2

c_double_p = C.POINTER(C.c_double)
vp = C.c_void_p


ABI_VERSION = 3


class _Sized(C.Structure):
    """Structs of the ABI carry their own size as the first member (the
    library rejects a caller whose layout differs from its own)."""

    def __init__(self, *args, **kw):
        super().__init__(*args, **kw)
        self.struct_size = C.sizeof(self)


class Lattice(_Sized):
    """pffmg_lattice (include/pffmg.h)."""
    _fields_ = [("struct_size", C.c_int32), ("dim", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("hx", C.c_double), ("hy", C.c_double), ("hz", C.c_double),
                ("n_vertices", C.c_int64),
                ("vrow_off", vp), ("vrow_lo", vp), ("vrow_hi", vp),
                ("crow_lo", vp), ("crow_hi", vp),
                ("own_lo", C.c_int32), ("own_hi", C.c_int32),
                ("plane0", C.c_int32), ("order", C.c_int32),
                ("tiles3d", vp), ("n_tiles3d", C.c_int32)]


class State(_Sized):
    """pffmg_state (include/pffmg.h)."""
    _fields_ = [("struct_size", C.c_int32), ("mu", C.c_double), ("lam", C.c_double), ("g_c", C.c_double),
                ("kappa", C.c_double), ("eps", C.c_double), ("pressure", C.c_double),
                ("split", C.c_int32), ("hints", C.c_int32),
                ("U", vp), ("phi_tilde", vp), ("rho", vp), ("flags", vp),
                ("split_band", C.c_double), ("phi_coef", vp)]


# name -> argtypes (restype is always c_int status unless noted)
_SIGS = {
    "pffmg_version": [],
    "pffmg_device_sm_count": [C.POINTER(C.c_int)],
    "pffmg_set_pdl": [C.c_int, C.POINTER(C.c_int)],
    "pffmg_apply": [C.POINTER(Lattice), C.POINTER(State), C.c_int, vp, vp, vp],
    "pffmg_residual": [C.POINTER(Lattice), C.POINTER(State), C.c_int, vp, vp, vp, vp],
    "pffmg_diagonal": [C.POINTER(Lattice), C.POINTER(State), vp, vp],
    "pffmg_phi_coef": [C.POINTER(Lattice), C.POINTER(State), vp, vp],
    "pffmg_semilinear_residual": [C.POINTER(Lattice), C.POINTER(State), vp, vp],
    "pffmg_cheb_step": [C.POINTER(Lattice), C.POINTER(State), C.c_int, vp, vp, vp, vp, vp,
                        C.c_double, C.c_double, C.c_int, vp],
    "pffmg_cheb_init": [C.POINTER(Lattice), C.POINTER(State), C.c_int, vp, vp, vp, vp, vp,
                        C.c_double, vp],
    "pffmg_apply_host": [C.POINTER(Lattice), C.POINTER(State), C.c_int, vp, vp, vp, vp, vp, C.c_int, vp],
    "pffmg_copy_h2d": [vp, vp, C.c_size_t, vp],
    "pffmg_copy_d2h": [vp, vp, C.c_size_t, vp],
    "pffmg_apply_pageable": [C.POINTER(Lattice), C.POINTER(State), C.c_int, vp, vp, vp, vp, vp, C.c_int, vp],
    "pffmg_qoi": [C.POINTER(Lattice), C.POINTER(State), C.c_int, vp, vp],
    "pffmg_boundary_load": [C.POINTER(Lattice), C.POINTER(State), vp, vp, C.c_int64, C.c_int, vp, vp, vp],
    "pffmg_coarse_cheb": [C.POINTER(Lattice), C.POINTER(State), vp, vp, vp, vp, vp, vp, C.c_int, vp, C.c_int, vp],
    "pffmg_cheb_step_bd": [C.POINTER(Lattice), C.POINTER(State), vp, vp, vp, vp, vp, vp, vp, C.c_int, vp],
    "pffmg_cheb_first_bd": [C.POINTER(Lattice), C.POINTER(State), vp, vp, vp, vp, vp, vp, vp, vp, vp],
    "pffmg_cheb_first_dc": [C.POINTER(Lattice), C.POINTER(State), C.c_int, vp, vp, vp, vp, vp, vp, vp, vp],
    "pffmg_cheb_init_bd": [C.POINTER(Lattice), C.POINTER(State), vp, vp, vp, vp, vp, vp, vp, vp],
    "pffmg_cheb_init_zero_bd": [vp, vp, vp, vp, C.c_int64, vp, vp, vp, C.c_int64, vp],
    "pffmg_cheb_step_dc": [C.POINTER(Lattice), C.POINTER(State), C.c_int, vp, vp, vp, vp, vp, vp,
                           C.c_int, vp],
    "pffmg_cheb_init_dc": [C.POINTER(Lattice), C.POINTER(State), C.c_int, vp, vp, vp, vp, vp, vp, vp],
    "pffmg_cheb_init_zero_dc": [vp, vp, vp, vp, vp, vp, C.c_int64, vp],
    "pffmg_jacobi_update_dc": [vp, vp, vp, vp, C.c_int64, vp],
    "pffmg_restrict": [C.POINTER(Lattice), C.POINTER(Lattice), C.c_int, C.c_int, vp, vp, vp, vp],
    "pffmg_restrict_init_bd": [C.POINTER(Lattice), C.POINTER(Lattice), vp, vp, vp, vp, vp, vp, vp, vp, vp, vp],
    "pffmg_prolongate": [C.POINTER(Lattice), C.POINTER(Lattice), C.c_int, C.c_int, vp, vp, vp,
                         C.c_int, vp],
    "pffmg_inject_f64": [C.POINTER(Lattice), C.POINTER(Lattice), C.c_int, vp, vp, vp],
    "pffmg_inject_flags": [C.POINTER(Lattice), C.POINTER(Lattice), vp, vp, vp],
    "pffmg_injection_map": [C.POINTER(Lattice), C.POINTER(Lattice), vp, vp],
    "pffmg_pack_flags": [vp, C.c_int, C.c_int64, vp, vp],
    "pffmg_unpack_flags": [vp, C.c_int, C.c_int64, vp, vp],
    "pffmg_masked_copy": [vp, C.c_int64, C.c_int, C.c_int, vp, vp, vp],
    "pffmg_masked_copy_init_bd": [vp, C.c_int64, C.c_int, vp, vp, vp, vp, vp, vp, vp, vp, vp],
    "pffmg_reciprocal": [vp, vp, C.c_int64, vp],
    "pffmg_cheb_init_zero": [vp, vp, C.c_double, vp, vp, vp, C.c_int64, vp],
    "pffmg_jacobi_update": [vp, vp, C.c_double, vp, C.c_int64, vp],
    "pffmg_axpy": [C.c_double, vp, vp, C.c_int64, vp],
    "pffmg_axpby": [C.c_double, vp, C.c_double, vp, C.c_int64, vp],
    "pffmg_scale": [C.c_double, vp, C.c_int64, vp],
    "pffmg_copy": [vp, vp, C.c_int64, vp],
    "pffmg_sub": [vp, vp, vp, C.c_int64, vp],
    "pffmg_dot": [vp, vp, C.c_int64, vp, vp],
    "pffmg_dot_scaled": [vp, vp, vp, C.c_int64, vp, vp],
    "pffmg_arnoldi_mgs": [vp, C.c_int64, C.c_int, vp, C.c_int64, vp, vp, vp],
    "pffmg_multi_axpy": [vp, C.c_int64, C.c_int, vp, vp, C.c_int64, vp],
    "pffmg_active_set": [vp, vp, vp, vp, C.c_double, vp, C.c_int, C.c_int64, vp, vp],
    "pffmg_cg_start": [vp, vp, vp, vp, vp, C.c_int64, vp, vp],
    "pffmg_cg_step": [vp, vp, vp, vp, vp, C.c_int64, vp, C.c_int, vp],
    "pffmg_dot_owned": [vp, vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, vp, vp],
    "pffmg_cg_dist": [C.c_int, vp, vp, vp, vp, vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, vp, vp],
    "pffmg_cg_dist_finish": [vp, C.c_int, vp],
    "pffmg_multi_dot_owned": [vp, C.c_int64, C.c_int, C.c_int, vp, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                              C.c_int64, vp, vp],
    "pffmg_gs_subtract": [vp, C.c_int64, C.c_int, vp, vp, C.c_int64, vp, C.c_int64, C.c_int64, C.c_int64, vp, vp],
    "pffmg_normalize": [vp, vp, C.c_int64, vp, vp, vp],
    "pffmg_pack_rows": [vp, C.c_int64, C.c_int, C.c_int64, C.c_int64, vp, C.c_int, vp],
}

_lib = None


class PffmgError(RuntimeError):
    """A libpffmg call returned a non-zero status."""


def load():
    """Load libpffmg.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise PffmgError(f"{LIB_PATH} not built: run `make -C {_HERE}/csrc` "
                             "(or __graft_entry__.build())")
        lib = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
        lib.pffmg_last_error.argtypes = []
        lib.pffmg_last_error.restype = C.c_char_p
        _lib = lib
    return _lib


def exported_symbols():
    return ["pffmg_last_error"] + list(_SIGS)


def call(name, *args):
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.pffmg_last_error().decode(errors="replace")
        raise PffmgError(f"{name} failed (status {rc}): {msg}")


def require_cuda():
    if not torch.cuda.is_available():
        raise PffmgError("pffmg needs a CUDA device (sm_100a); there is no CPU fallback")
    load()


_DEVICE = None


def stream():
    """Current torch stream as a cudaStream_t.  libpffmg keeps per-process
    launch caches (occupancy, cooperative-grid scratch) for the device it was
    first used on, so one process drives one device (one rank per GPU)."""
    global _DEVICE
    d = torch.cuda.current_device()
    if _DEVICE is None:
        _DEVICE = d
    elif d != _DEVICE:
        raise PffmgError(f"libpffmg was first used on cuda:{_DEVICE} in this process; "
                         f"cuda:{d} needs its own process (one rank per GPU)")
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    """Device pointer of a tensor (or None)."""
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())

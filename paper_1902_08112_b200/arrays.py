"""Host/device array plumbing shared by the drop-in twins.

Public entry points accept numpy arrays or CUDA tensors and return the kind
they were given; internally every vector is a float64 CUDA tensor.
Callables supplied by users (operators, preconditioners) receive CUDA
tensors; a callable that cannot take one (it raises TypeError, e.g. a plain
numpy matrix product) is switched to numpy in/out transparently -- that only
moves the user's own data, never the pffmg kernels, to the host.
"""
from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib

F64 = torch.float64


def is_tensor(a):
    return isinstance(a, torch.Tensor)


# large numpy arrays cross the link through libpffmg's
# threaded page-locked staging (pffmg_copy_h2d / _d2h) instead of the driver's
# single-threaded pageable copy (PFFMG_THREADED_COPIES=0: plain torch copies)
THREADED_COPIES = os.environ.get("PFFMG_THREADED_COPIES", "1") != "0"
# measured on the B200 hosts (tools/copybench.py): host -> device beats torch's
# pageable copy from ~16 MiB on (28 vs 21 GB/s at 25 MB, 37 vs 12 at 100 MB; below,
# the pool threads' wake-up costs more than it saves), device -> host from a few
# MiB on (30 vs 17 GB/s at 8 MB, 46 vs 18 at 25 MB, 40 vs 2 at 100 MB)
THREADED_MIN_H2D = 16 << 20
THREADED_MIN_D2H = 4 << 20


def dev(a, dtype=F64):
    """float64 (or dtype) contiguous CUDA tensor view/copy of `a`."""
    if isinstance(a, torch.Tensor):
        if not a.is_cuda:
            a = a.to("cuda", non_blocking=False)
        if a.dtype != dtype:
            a = a.to(dtype)
        return a.contiguous()
    arr = np.ascontiguousarray(np.asarray(a), dtype=_np_dtype(dtype))
    if THREADED_COPIES and arr.nbytes >= THREADED_MIN_H2D:
        out = torch.empty(arr.shape, dtype=dtype, device="cuda")
        _lib.call("pffmg_copy_h2d", arr.ctypes.data, _lib.ptr(out), arr.nbytes, _lib.stream())
        return out
    return torch.from_numpy(arr).to("cuda")


_NP_OF = {torch.float64: np.float64, torch.uint8: np.uint8, torch.bool: np.bool_,
          torch.int64: np.int64, torch.int32: np.int32}


def _np_dtype(dtype):
    return _NP_OF[dtype]


def copy_into(buf, src, dtype=F64):
    """buf (a contiguous CUDA tensor) <- src (tensor or numpy array of the same size)."""
    if isinstance(src, torch.Tensor):
        buf.copy_(src)
        return buf
    arr = np.ascontiguousarray(np.asarray(src), dtype=_np_dtype(dtype))
    if arr.size != buf.numel():
        raise ValueError(f"expected {buf.numel()} entries, got {arr.size}")
    if THREADED_COPIES and arr.nbytes >= THREADED_MIN_H2D and buf.is_contiguous() and buf.dtype == dtype:
        _lib.call("pffmg_copy_h2d", arr.ctypes.data, _lib.ptr(buf), arr.nbytes, _lib.stream())
    else:
        buf.copy_(torch.from_numpy(arr).reshape(buf.shape))
    return buf


def host(t):
    t = t.detach()
    nbytes = t.numel() * t.element_size()
    if THREADED_COPIES and t.is_cuda and nbytes >= THREADED_MIN_D2H and t.dtype in _NP_OF:
        t = t.contiguous()
        out = np.empty(tuple(t.shape), dtype=_NP_OF[t.dtype])
        _lib.call("pffmg_copy_d2h", _lib.ptr(t), out.ctypes.data, nbytes, _lib.stream())
        return out
    return t.cpu().numpy()


def like(out, ref, dst=None):
    """Return `out` (CUDA tensor) as the kind of `ref`: numpy -> numpy copy,
    CPU tensor -> CPU tensor, CUDA tensor -> itself.  With `dst` given
    (numpy array or tensor of the right size) the result is written into it."""
    if dst is not None:
        if isinstance(dst, torch.Tensor):
            dst.copy_(out, non_blocking=dst.is_pinned())
            if dst.is_pinned():
                torch.cuda.current_stream().synchronize()
        else:
            np.copyto(dst, host(out))
        return dst
    if isinstance(ref, torch.Tensor):
        return out if ref.is_cuda else out.cpu()
    return host(out)


def empty(n, dtype=F64):
    return torch.empty(int(n), dtype=dtype, device="cuda")


def zeros(n, dtype=F64):
    return torch.zeros(int(n), dtype=dtype, device="cuda")


class DeviceCallable:
    """Wrap a user callable so it can be fed CUDA tensors; falls back to numpy
    in/out for callables that only understand numpy."""

    def __init__(self, fn):
        self.fn = fn
        self.numpy_mode = getattr(fn, "_pffmg_numpy_only", False)

    def __call__(self, v):
        if not self.numpy_mode:
            try:
                out = self.fn(v)
            except (_lib.PffmgError, torch.cuda.OutOfMemoryError):
                raise
            except (TypeError, RuntimeError) as e:
                # only a numpy-only callable (e.g. `lambda v: A @ v` with a numpy A)
                # switches to host round trips; CUDA failures propagate
                if not _is_numpy_conversion_error(e):
                    raise
                self.numpy_mode = True
            else:
                return dev(out)
        return dev(self.fn(host(v)))


_CONVERSION_HINTS = ("numpy", "ndarray", "can't convert", "cannot convert", "__array__")


def _is_numpy_conversion_error(e):
    """True for the errors a numpy-only callable raises when handed a CUDA
    tensor (TypeError from numpy's conversion, or torch refusing an ndarray)."""
    msg = str(e)
    if "CUDA" in msg and "error" in msg.lower():
        return False
    return isinstance(e, TypeError) or any(h in msg for h in _CONVERSION_HINTS)


def pack_flags(mask_bool, n_comp, V):
    """Packed per-vertex constraint bits from a bool[n_comp*V] mask."""
    m = dev(mask_bool, torch.uint8) if not (is_tensor(mask_bool) and mask_bool.dtype == torch.bool) \
        else mask_bool.to(torch.uint8).contiguous()
    if m.numel() != n_comp * V:
        raise ValueError(f"mask has {m.numel()} entries, expected {n_comp * V}")
    out = flags_buffer(V)
    _lib.call("pffmg_pack_flags", _lib.ptr(m), n_comp, V, _lib.ptr(out), _lib.stream())
    return out


def unpack_flags(flags, n_comp, V):
    out = empty(n_comp * V, torch.uint8)
    _lib.call("pffmg_unpack_flags", _lib.ptr(flags), n_comp, V, _lib.ptr(out), _lib.stream())
    return out.to(torch.bool)


class DeviceScalar:
    """Small device scratch array for reductions."""

    def __init__(self, n=1):
        self.t = torch.zeros(n, dtype=F64, device="cuda")

    def ptr(self, i=0):
        import ctypes
        return ctypes.c_void_p(self.t.data_ptr() + 8 * i)

    def item(self, i=0):
        return float(self.t[i].item())


def dot(x, y, out=None, offset=0):
    """Deterministic device dot product; returns the DeviceScalar holding it."""
    s = out or DeviceScalar()
    _lib.call("pffmg_dot", _lib.ptr(x), _lib.ptr(y), x.numel(), s.ptr(offset), _lib.stream())
    return s


def norm(x):
    return float(np.sqrt(dot(x, x).item()))


FLAG_PAD = 64


def flags_buffer(V):
    """Packed-flag buffer of V bytes; the kernels read flags as aligned 32-bit
    words, so the allocation is padded (include/pffmg.h) and the pad zeroed."""
    buf = torch.zeros(int(V) + FLAG_PAD, dtype=torch.uint8, device="cuda")
    return buf[:int(V)]

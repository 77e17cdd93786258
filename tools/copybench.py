"""Pageable host <-> device copy bandwidth: libpffmg's threaded staging
(pffmg_copy_h2d / _d2h) against torch's pageable copies, by size."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08112_b200 import _lib, arrays  # noqa: E402


def med(fn, reps=9):
    fn(); fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


for mb in (8, 25, 100):
    n = mb * (1 << 20) // 8
    a = np.random.default_rng(0).standard_normal(n)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    out = np.empty(n)
    pin = torch.from_numpy(a).pin_memory()
    t_pin = med(lambda: d.copy_(pin, non_blocking=True))
    t_torch = med(lambda: d.copy_(torch.from_numpy(a)))
    t_thr = med(lambda: _lib.call("pffmg_copy_h2d", a.ctypes.data, _lib.ptr(d), a.nbytes, _lib.stream()))
    t_back_torch = med(lambda: d.cpu())
    t_back_thr = med(lambda: _lib.call("pffmg_copy_d2h", _lib.ptr(d), out.ctypes.data, a.nbytes, _lib.stream()))
    t_memcpy = med(lambda: np.copyto(out, a))
    g = lambda t: a.nbytes / t * 1e-9  # noqa: E731
    print(f"== {mb} MB threads={os.environ.get('PFFMG_COPY_THREADS', 'default')}: h2d pinned {g(t_pin):.1f} torch-pageable "
          f"{g(t_torch):.1f} threaded {g(t_thr):.1f} GB/s | d2h torch {g(t_back_torch):.1f} threaded {g(t_back_thr):.1f} GB/s"
          f" | host memcpy 1 thread {g(t_memcpy):.1f} GB/s", flush=True)

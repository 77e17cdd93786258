"""pffmg_apply_host strip-count sweep on cfg2 (pinned host in/out)."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08112_b200 import _lib, configs  # noqa: E402
from paper_1902_08112_b200.model import ConstraintMask, PhaseFieldOperator, SplitKind  # noqa: E402

prob = configs.make("cfg2")
mask = prob.dirichlet.combined_with(prob.active, np.zeros(prob.n_dofs))
op = PhaseFieldOperator(prob.disc.finest, prob.state, ConstraintMask(mask.is_constrained, mask.inhomogeneity),
                        prob.params, SplitKind.NOSPLIT)
n = op.n_dofs
v = torch.from_numpy(prob.v.copy()).pin_memory()
out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in, d_out = torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64, device="cuda")


def run(strips):
    _lib.call("pffmg_apply_host", op.lat.ref, op._stp, _lib.FULL, ctypes.c_void_p(v.data_ptr()),
              ctypes.c_void_p(out.data_ptr()), _lib.ptr(d_in), _lib.ptr(d_out), None, strips, _lib.stream())
    torch.cuda.current_stream().synchronize()


for strips in (4, 6, 8, 12):
    run(strips)
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        run(strips)
        ts.append(time.perf_counter() - t0)
    t = float(np.median(ts))
    print(f"strips {strips:3d}: {t * 1e3:.3f} ms  {n / t * 1e-9:.2f} GDoF/s")

if len(sys.argv) > 1:
    from torch.profiler import ProfilerActivity, profile
    k = int(sys.argv[1])
    run(k)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        run(k)
    ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    for e in ev:
        print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f}  {e.name[:50]}")

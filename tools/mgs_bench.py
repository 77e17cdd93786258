"""Time one Arnoldi step (pffmg_arnoldi_mgs) at the cfg2 size for j = 0..12
(PFFMG_MGS_COOP=0 selects the multi-launch sweep)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1902_08112_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_151_875
m = 30
V = torch.randn((m + 1, n), dtype=torch.float64, device="cuda")
V /= V.norm(dim=1, keepdim=True)
w0 = torch.randn(n, dtype=torch.float64, device="cuda")
h = torch.zeros(m + 1, dtype=torch.float64, device="cuda")
ctl = torch.zeros(67, dtype=torch.float64, device="cuda")
tot = 0.0
for j in (0, 3, 6, 9, 12):
    def step():
        V[j + 1].copy_(w0)
        _lib.call("pffmg_arnoldi_mgs", _lib.ptr(V), V.stride(0), j, _lib.ptr(V[j + 1]), n, _lib.ptr(h),
                  _lib.ptr(ctl), _lib.stream())
    for _ in range(3):
        step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    c0.record()
    for _ in range(reps):
        V[j + 1].copy_(w0)
    c1.record()
    torch.cuda.synchronize()
    t = (e0.elapsed_time(e1) - c0.elapsed_time(c1)) / reps * 1e3
    print(f"j={j:2d}: {t:7.1f} us per Arnoldi step")

"""Anatomy of one replayed V-cycle: kernel durations, gaps, per-level split.

    python tools/prof_vcycle.py [config]
"""
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08112_b200 import configs, mgsolve, model as M  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
prob = configs.make(name)
ctxs = mgsolve.build_level_contexts(prob.disc, prob.state, prob.active, prob.dirichlet, prob.params,
                                    M.SplitKind.NOSPLIT)
r = torch.randn(ctxs[-1].op.n_dofs, dtype=torch.float64, device="cuda")
pc = mgsolve.VCyclePreconditioner(ctxs, degree=prob.degree)
out = torch.empty_like(r)
for _ in range(3):
    pc._pffmg_into(r, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(20):
    e0.record()
    pc._pffmg_into(r, out)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"vcycle replay: median {np.median(ts) * 1e3:.1f} us  min {min(ts) * 1e3:.1f} us")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    pc._pffmg_into(r, out)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
busy = sum(e.time_range.end - e.time_range.start for e in ev)
span = ev[-1].time_range.end - ev[0].time_range.start
print(f"kernels {len(ev)}  busy {busy:.1f} us  span {span:.1f} us  gaps {span - busy:.1f} us")
# group by grid-size class: the fine level kernels are the long ones
rows = {}
for e in ev:
    d = e.time_range.end - e.time_range.start
    k = e.name[:60]
    a = rows.setdefault(k, [0, 0.0, []])
    a[0] += 1
    a[1] += d
    a[2].append(d)
for k, (n, t, ds) in sorted(rows.items(), key=lambda kv: -kv[1][1]):
    print(f"{t:9.1f} us {n:4d}x  max {max(ds):7.1f}  min {min(ds):6.1f}  {k}")
short = [e.time_range.end - e.time_range.start for e in ev]
print("kernels < 5 us:", sum(1 for d in short if d < 5), "total", sum(d for d in short if d < 5))
if os.environ.get("PFFMG_VC_SEQ"):
    for e in ev:
        print(f"{e.time_range.start - ev[0].time_range.start:9.1f} {e.time_range.end - e.time_range.start:7.1f}  {e.name[:70]}")

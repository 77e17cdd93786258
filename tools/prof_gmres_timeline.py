"""GPU timeline of one GMRES solve (after the setup): busy time, idle gaps
and the kernels that follow each gap (host-side stalls show up as gaps)."""
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08112_b200 import configs, krylov, mgsolve, model as M  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
prob = configs.make(name)
rhs = torch.as_tensor(configs.fallback_rhs(prob), device="cuda")
ctxs = mgsolve.build_level_contexts(prob.disc, prob.state, prob.active, prob.dirichlet, prob.params,
                                    M.SplitKind.NOSPLIT)
ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8)
pc = mgsolve.VCyclePreconditioner(ctxs, degree=prob.degree)
for _ in range(2):
    krylov.gmres(ctxs[-1].op.apply, pc, rhs, ctl)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    x, its = krylov.gmres(ctxs[-1].op.apply, pc, rhs, ctl)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
span = ev[-1].time_range.end - t0
busy = sum(e.time_range.end - e.time_range.start for e in ev)
print(f"its {its}  kernels {len(ev)}  span {span:.0f} us  busy {busy:.0f} us")
gaps = []
end = ev[0].time_range.end
prev = ev[0].name
for e in ev[1:]:
    g = e.time_range.start - end
    if g > 3:
        gaps.append((g, e.name[:60], e.time_range.start - t0))
        if g > 50:
            print(f"gap {g:7.0f} us at {e.time_range.start - t0:8.0f}: after {prev[:50]} -> before {e.name[:50]}")
    end = max(end, e.time_range.end)
    prev = e.name
tot = sum(g for g, _, _ in gaps)
print(f"gaps > 3 us: {len(gaps)}  total {tot:.0f} us")
by = {}
for g, n, _ in gaps:
    a = by.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += g
for n, (c, t) in sorted(by.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"  {t:8.0f} us over {c:3d} gaps before {n}")
cat = {}
for e in ev:
    k = e.name[:40]
    cat[k] = cat.get(k, 0.0) + (e.time_range.end - e.time_range.start)
for k, t in sorted(cat.items(), key=lambda kv: -kv[1])[:12]:
    print(f"  {t:8.0f} us  {k}")

import cProfile  # noqa: E402
import pstats  # noqa: E402
import time  # noqa: E402
torch.cuda.synchronize()
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
krylov.gmres(ctxs[-1].op.apply, pc, rhs, ctl)
torch.cuda.synchronize()
pr.disable()
print("gmres wall", time.perf_counter() - t)
pstats.Stats(pr).sort_stats("tottime").print_stats(12)

# which host calls stall the start of a solve?
_orig_ws, _orig_zeros, _orig_norm = krylov._workspace, krylov.zeros, krylov.norm


def _timed(name, fn):
    def w(*a, **k):
        t = time.perf_counter()
        r = fn(*a, **k)
        print(f"  {name}: {1e3 * (time.perf_counter() - t):.3f} ms")
        return r
    return w


krylov._workspace = _timed("_workspace", _orig_ws)
krylov.zeros = _timed("zeros", _orig_zeros)
krylov.norm = _timed("norm", _orig_norm)
torch.cuda.synchronize()
krylov.gmres(ctxs[-1].op.apply, pc, rhs, ctl)
torch.cuda.synchronize()

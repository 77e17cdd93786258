"""Time the pieces of one Newton-step linear solve at cfg2 (host-side view)."""
import cProfile
import pstats
import sys
import os
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08112_b200 import configs, krylov, mgsolve  # noqa: E402
from paper_1902_08112_b200.model import SplitKind  # noqa: E402

prob = configs.make(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
rhs = torch.as_tensor(configs.fallback_rhs(prob), device="cuda")


from paper_1902_08112_b200 import model as M  # noqa: E402

# the state as a Newton loop holds it: on the device (bench.py newton_step)
state_dev = M.LinearizationState(
    U=torch.as_tensor(prob.state.U, device="cuda"), U_prev1=torch.as_tensor(prob.state.U_prev1, device="cuda"),
    U_prev2=torch.as_tensor(prob.state.U_prev2, device="cuda"), t=prob.state.t,
    t_prev1=prob.state.t_prev1, t_prev2=prob.state.t_prev2,
    phi_tilde=torch.as_tensor(prob.state.phi_tilde, device="cuda"))


def setup():
    return mgsolve.build_level_contexts(prob.disc, state_dev, prob.active, prob.dirichlet,
                                        prob.params, SplitKind.NOSPLIT)


ctxs = setup()
torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter()
    ctxs = setup()
    torch.cuda.synchronize()
    print("setup", time.perf_counter() - t0)
pr = cProfile.Profile()
pr.enable()
ctxs = setup()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
pc = mgsolve.VCyclePreconditioner(ctxs, degree=prob.degree)
ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8)
x, its = krylov.gmres(ctxs[-1].op.apply, pc, rhs, ctl)
torch.cuda.synchronize()
t0 = time.perf_counter()
x, its = krylov.gmres(ctxs[-1].op.apply, pc, rhs, ctl)
torch.cuda.synchronize()
print("gmres", its, time.perf_counter() - t0)
t0 = time.perf_counter()
for _ in range(10):
    pc._pffmg_into(rhs, x)
torch.cuda.synchronize()
print("vcycle", (time.perf_counter() - t0) / 10)
# device time of one setup-graph replay
sess = ctxs[-1]._session
if sess is not None and sess.graph is not None:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        e0.record()
        sess.graph.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print("setup graph replay ms", sorted(ts)[5])
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        sess.graph.replay()
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14))

"""Where does one Newton-step solve spend its time?  Wall clock of setup and
GMRES vs the summed device time of the kernels (torch.profiler / CUPTI)."""
import os
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08112_b200 import configs, krylov, mgsolve, model as M  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
prob = configs.make(name)
mask = prob.dirichlet.combined_with(prob.active, prob.active * 0.0)
cm = torch.as_tensor(mask.is_constrained, device="cuda")
st = M.LinearizationState(U=torch.as_tensor(prob.state.U, device="cuda"),
                          U_prev1=torch.as_tensor(prob.state.U_prev1, device="cuda"),
                          U_prev2=torch.as_tensor(prob.state.U_prev2, device="cuda"), t=0.0, t_prev1=0.0,
                          t_prev2=0.0, phi_tilde=torch.as_tensor(prob.state.phi_tilde, device="cuda"))
ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8)


def step():
    t0 = time.perf_counter()
    R = M.residual(prob.disc.finest, st, prob.dirichlet, prob.params, M.SplitKind.NOSPLIT)
    R.neg_()
    R[cm] = 0
    torch.cuda.synchronize()
    print("  residual", time.perf_counter() - t0)
    ctxs = mgsolve.build_level_contexts(prob.disc, st, prob.active, prob.dirichlet, prob.params,
                                        M.SplitKind.NOSPLIT)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pc = mgsolve.VCyclePreconditioner(ctxs, degree=prob.degree)
    x, its = krylov.gmres(ctxs[-1].op.apply, pc, R, ctl)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1, its


step()
print("wall", step())
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    res = step()
print("profiled wall", res)
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
tot = sum(e.device_time for e in ev)
print(f"kernels {len(ev)}  device time {tot / 1e3:.2f} ms")
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))

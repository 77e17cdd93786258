"""Wall-clock anatomy of one bench.py Newton step (cfg2 by default): residual
RHS, build_level_contexts (setup graph + spectra), GMRES, with syncs between
the phases so each number is that phase alone."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08112_b200 import configs, krylov, mgsolve, model as M  # noqa: E402
from paper_1902_08112_b200.model import SplitKind  # noqa: E402

prob = configs.make(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
mask = prob.dirichlet.combined_with(prob.active, np.zeros(prob.n_dofs))
cmask_dev = torch.as_tensor(mask.is_constrained, device="cuda")
state_dev = M.LinearizationState(
    U=torch.as_tensor(prob.state.U, device="cuda"), U_prev1=torch.as_tensor(prob.state.U_prev1, device="cuda"),
    U_prev2=torch.as_tensor(prob.state.U_prev2, device="cuda"), t=prob.state.t,
    t_prev1=prob.state.t_prev1, t_prev2=prob.state.t_prev2,
    phi_tilde=torch.as_tensor(prob.state.phi_tilde, device="cuda"))
DEVMASK = os.environ.get("DEVMASK", "1") == "1"
if DEVMASK:   # masks held on the device by the Newton loop, like the state
    dirichlet = M.ConstraintMask(torch.as_tensor(prob.dirichlet.is_constrained, device="cuda"),
                                 torch.as_tensor(prob.dirichlet.inhomogeneity, device="cuda"))
    active = torch.as_tensor(prob.active, device="cuda")
else:
    dirichlet, active = prob.dirichlet, prob.active
ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)


def step(sync):
    t = [time.perf_counter()]
    R = M.residual(prob.disc.finest, state_dev, dirichlet, prob.params, SplitKind.NOSPLIT)
    if sync:
        torch.cuda.synchronize()
    t.append(time.perf_counter())
    R.neg_()
    R[cmask_dev] = 0.0
    if sync:
        torch.cuda.synchronize()
    t.append(time.perf_counter())
    ctxs = mgsolve.build_level_contexts(prob.disc, state_dev, active, dirichlet,
                                        prob.params, SplitKind.NOSPLIT)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    pc = mgsolve.VCyclePreconditioner(ctxs, degree=prob.degree)
    x, its = krylov.gmres(ctxs[-1].op.apply, pc, R, ctl)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    return np.diff(t) * 1e3, its, x


x_ref = step(False)[2].clone()
print("iterations", step(False)[1])
for sync in (False, True):
    step(sync)
    rs = np.array([step(sync)[0] for _ in range(5)])
    med = np.median(rs, axis=0)
    print(f"sync={sync}: residual {med[0]:.3f} ms  neg+mask {med[1]:.3f}  build {med[2]:.3f}  gmres {med[3]:.3f}"
          f"  total {med.sum():.3f}")

import cProfile, pstats  # noqa: E401,E402
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    step(False)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

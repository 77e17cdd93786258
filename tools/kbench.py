"""Kernel microbenchmark: time one operator mode on a config (CUDA events,
L2 flushed between reps).  Used for tuning and under ncu."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08112_b200 import _lib, configs  # noqa: E402
from paper_1902_08112_b200.model import ConstraintMask, PhaseFieldOperator, SplitKind  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--levels", type=int, default=None)
ap.add_argument("--mode", default="full", choices=["full", "u", "phi", "diag", "chebu", "chebp", "resid", "chebbd", "initbd"])
ap.add_argument("--reps", type=int, default=200)
ap.add_argument("--pre", action="store_true", help="use the pre-masked hint (inputs zeroed at constraints)")
args = ap.parse_args()

prob = configs.make(args.config, args.levels)
mask = prob.dirichlet.combined_with(prob.active, np.zeros(prob.n_dofs))
op = PhaseFieldOperator(prob.disc.finest, prob.state, ConstraintMask(mask.is_constrained, mask.inhomogeneity),
                        prob.params, SplitKind.NOSPLIT)
n, d, V = op.n_dofs, op.dim * op.V, op.V
v = torch.as_tensor(prob.v, device="cuda")
if args.pre:
    v[torch.as_tensor(mask.is_constrained, device="cuda")] = 0.0
P = args.pre
out = torch.empty_like(v)
r = torch.randn(n, dtype=torch.float64, device="cuda")
x = torch.randn(n, dtype=torch.float64, device="cuda")
inv = torch.rand(n, dtype=torch.float64, device="cuda") + 1.0
d2 = torch.empty_like(v)
cf = torch.tensor([0.3, 0.2], dtype=torch.float64, device="cuda")
flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")


def run():
    if args.mode == "full":
        op.apply_dev(_lib.FULL, v, out, pre=P)
    elif args.mode == "u":
        op.apply_dev(0, v[:d], out[:d], pre=P)
    elif args.mode == "phi":
        op.apply_dev(1, v[d:], out[d:], pre=P)
    elif args.mode == "diag":
        op.diagonal_dev(out)
    elif args.mode == "resid":
        op.residual_dev(_lib.FULL, v, r, out, pre=P)
    elif args.mode == "chebu":
        op.cheb_step_dev(0, v[:d], d2[:d], r[:d], x[:d], inv[:d], 0.3, 0.2, pre=P)
    elif args.mode == "chebbd":      # the block-diagonal smoother step of the V-cycle
        op.cheb_step_bd(v, d2, r, x, inv, cf, cf, pre=P)
    elif args.mode == "initbd":      # its first step from a non-zero x (r = b - A x)
        op.cheb_init_bd(x, v, r, d2, inv, cf[:1], cf[:1], pre=P)
    elif args.mode == "chebp":
        op.cheb_step_dev(1, v[d:], d2[d:], r[d:], x[d:], inv[d:], 0.3, 0.2, pre=P)


for _ in range(3):
    flush.zero_()
    run()
torch.cuda.synchronize()
ts = []
for _ in range(args.reps):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ndof = {"full": n, "resid": n, "diag": n, "chebbd": n, "initbd": n, "u": d, "chebu": d, "phi": V, "chebp": V}[args.mode]
# the event timer ticks in ~2 us steps on these boxes: the mean over many reps
# resolves below a tick, the median does not
print(f"{args.config} {args.mode}{' pre' if P else ''}: mean {np.mean(ts)*1e3:.2f} us  median {np.median(ts)*1e3:.1f} us  "
      f"{ndof / np.mean(ts) * 1e-6:.1f} GDoF/s")

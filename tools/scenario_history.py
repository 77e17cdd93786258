"""Per-iteration active-set history of the first step of a golden scenario,
run by the reference (unpatched) or with the GPU twins installed (--patched).
Debug aid for tests/test_gpu_patch.py."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(p, "fracmg")):
        sys.path.insert(0, p)
        break
from fracmg import nonlinear, scenarios  # noqa: E402

from tests.golden.make_golden_specs import scenario  # noqa: E402

tag = sys.argv[1]
patched = "--patched" in sys.argv
if patched:
    import fracmg

    from paper_1902_08112_b200 import patch
    patch.install(fracmg, operator=True, physics=True)
orig = nonlinear.ActiveSetSolver.solve_step
log = []


def traced(self, state, dirichlet, phi_old, active_prev=None):
    U, rep, active = orig(self, state, dirichlet, phi_old, active_prev)
    log.append([(h.set_size, h.set_changed, h.residual_norm, h.gmres_iters) for h in rep.history])
    return U, rep, active


nonlinear.ActiveSetSolver.solve_step = traced
sc = scenario(scenarios, tag)
from dataclasses import replace  # noqa: E402
sc = replace(sc, t_end=sc.dt)
scenarios.run(sc)
for step in log:
    for h in step:
        print(h)

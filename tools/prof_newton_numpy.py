"""cProfile of the numpy-I/O Newton step of bench.py (solve.numpy_io): where the
host time of the reference driver's calling convention goes."""
import cProfile
import os
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1902_08112_b200 import configs  # noqa: E402

prob = configs.make(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
mask = prob.dirichlet.combined_with(prob.active, np.zeros(prob.n_dofs))
step = bench.newton_step_numpy_fn(prob, mask)
for _ in range(3):
    print("step %.2f ms" % (step()[0] * 1e3))
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)

"""Stress of the threaded host paths (pool wake-ups, piece claiming, ring-slot
recycling): random sizes and directions, contents checked every time; then the
pageable apply against the device apply on two lattices.  Run under `timeout`."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08112_b200 import _lib, arrays, configs, model  # noqa: E402
from paper_1902_08112_b200.model import ConstraintMask, PhaseFieldOperator, SplitKind  # noqa: E402

rng = np.random.default_rng(int(os.environ.get("SEED", "0")))
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
big = rng.standard_normal(16 << 20)            # 128 MB of doubles
dbig = torch.from_numpy(big).cuda()
out = np.empty_like(big)
t0 = time.time()
for it in range(iters):
    nb = int(rng.choice([8, 4096, (4 << 20) - 8, 4 << 20, (4 << 20) + 8, int(rng.integers(1, 16 << 20)) * 8]))
    n = nb // 8
    o = int(rng.integers(0, big.size - n + 1))
    if rng.random() < 0.5:
        d = torch.empty(n, dtype=torch.float64, device="cuda")
        _lib.call("pffmg_copy_h2d", big[o:o + n].ctypes.data, _lib.ptr(d), nb, _lib.stream())
        assert torch.equal(d, dbig[o:o + n]), ("h2d", it, nb)
    else:
        out[:n] = np.nan
        _lib.call("pffmg_copy_d2h", _lib.ptr(dbig[o:o + n]), out.ctypes.data, nb, _lib.stream())
        assert np.array_equal(out[:n], big[o:o + n]), ("d2h", it, nb)
    if it % 7 == 0:
        time.sleep(float(rng.random()) * 2e-3)   # let the pool park between calls
print(f"copies ok: {iters} in {time.time() - t0:.1f} s", flush=True)

model.PAGEABLE_MIN = 1
for cfg, reps in (("cfg1", 400), ("cfg4", 60)):
    prob = configs.make(cfg)
    mask = prob.dirichlet.combined_with(prob.active, np.zeros(prob.n_dofs))
    op = PhaseFieldOperator(prob.disc.finest, prob.state, ConstraintMask(mask.is_constrained, mask.inhomogeneity),
                            prob.params, SplitKind.NOSPLIT)
    v = prob.v.copy()
    ref = op.apply(torch.as_tensor(v).cuda()).cpu().numpy()
    for it in range(reps):
        got = op.apply(v)
        assert np.array_equal(got, ref), (cfg, it)
        if it % 5 == 0:
            time.sleep(float(rng.random()) * 2e-3)
    print(f"pageable apply ok: {cfg} x{reps}", flush=True)

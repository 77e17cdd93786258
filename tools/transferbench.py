import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1902_08112_b200 import _lib, configs, mgsolve, model as M
for cfg, lv in (("cfg4", None), ("cfg5", 7), ("cfg2", None)):
    prob = configs.make(cfg, lv)
    D = prob.disc
    from paper_1902_08112_b200.fem import Discretization
    D = Discretization.wrap(D)
    L = D.hierarchy.n_levels
    nc = D.hierarchy.dim + 1
    Vf, Vc = D.hierarchy.levels[-1].n_vertices, D.hierarchy.levels[-2].n_vertices
    xf = torch.randn(nc * Vf, dtype=torch.float64, device="cuda"); xc = torch.randn(nc * Vc, dtype=torch.float64, device="cuda")
    ff = torch.zeros(Vf + 64, dtype=torch.uint8, device="cuda")[:Vf]; fc = torch.zeros(Vc + 64, dtype=torch.uint8, device="cuda")[:Vc]
    flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
    def t(fn, reps=20):
        fn(); torch.cuda.synchronize(); ts = []
        for _ in range(reps):
            flush.zero_(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        return np.median(ts) * 1e3
    tp = t(lambda: D.prolongate_dev(xc, xf, L - 2, nc, 0, ff, accumulate=True))
    tr = t(lambda: D.restrict_dev(xf, xc, L - 2, nc, 0, fc))
    bp = (2 * nc * Vf + nc * Vc) * 8; br = (nc * Vf + nc * Vc) * 8
    print(f"== {cfg} Vf={Vf}: prolongate {tp:.1f} us ({bp / tp * 1e-6:.0f} GB/s)  restrict {tr:.1f} us ({br / tr * 1e-6:.0f} GB/s)", flush=True)

"""Debug: which mode / vertices differ between non-PRE, PRE and a repeat (Miehe, cfg1 golden)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from tests.conftest import Golden
from tests.test_gpu_miehe import _case
from paper_1902_08112_b200 import _lib
from paper_1902_08112_b200 import model as M
g = {n: Golden(n) for n in ("operator_band",)}
for name in sys.argv[1:] or ["cfg1"]:
    gg, tag, space, st, mask, params = _case(g, name, "operator_band", "masked")
    for split in (M.SplitKind.MIEHE, M.SplitKind.NOSPLIT):
        op = M.PhaseFieldOperator(space, st, mask, params, split)
        flags = torch.as_tensor(gg[f"{tag}/flags"], device="cuda")
        v = torch.as_tensor(gg[f"{tag}/v"], device="cuda").clone()
        v[flags] = 0.0
        d = op.dim * op.V
        nx = int(round(np.sqrt(op.V))) - 1
        for which, vin, n in ((_lib.FULL, v, op.n_dofs), (0, v[:d], d), (1, v[d:], op.V)):
            a = torch.empty(n, dtype=torch.float64, device="cuda"); b = torch.empty_like(a); c = torch.empty_like(a)
            op.apply_dev(which, vin, a); op.apply_dev(which, vin, b, pre=True); op.apply_dev(which, vin, c)
            for lbl, x in (("pre", b), ("repeat", c)):
                bad = torch.nonzero(a != x).flatten().cpu().numpy()
                if bad.size:
                    vv = bad % op.V
                    print(name, split, which, lbl, bad.size, "V", op.V, "x", (vv % (nx + 1))[:20], "y", (vv // (nx + 1))[:20],
                          "maxdiff", float((a - x).abs().max()))
                else:
                    print(name, split, which, lbl, "equal")

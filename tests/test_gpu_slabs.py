"""The CUDA operator on slab sub-lattices (own_lo/own_hi): every rank's
owned rows, computed from its slab with ghost planes filled from the global
vector, must stitch to the single-GPU result.  Ranks are emulated one after
another in one process (no inter-rank waiting); the communication layer is
covered by tests/test_distributed_cpu.py."""
import numpy as np
import pytest
import torch

from tests.conftest import rel_err
from tests.golden.specs import MESHES

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,world", [("cfg1", 2), ("cfg1", 5), ("cube", 2), ("lprism", 2),
                                        ("rect3d", 3), ("lshape3d", 2)])
def test_slab_operator_stitches(name, world):
    from paper_1902_08112_b200 import _lib, distributed as D, lattice
    from paper_1902_08112_b200.fem import Discretization, build_hierarchy
    from paper_1902_08112_b200.model import ConstraintMask, LinearizationState, MaterialParams, \
        PhaseFieldOperator, SplitKind
    blocks, n_levels, dim = MESHES[name]
    n_levels += 1
    disc = Discretization(build_hierarchy(blocks, n_levels, dim))
    levels = disc.hierarchy.levels
    fine = levels[-1]
    V = fine.n_vertices
    n = (dim + 1) * V
    rng = np.random.default_rng(11)
    U = 1e-2 * rng.standard_normal(n)
    U[dim * V:] = np.clip(0.6 + 0.4 * rng.standard_normal(V), 0, 1)
    st = LinearizationState(U=U, U_prev1=U, U_prev2=U, t=0.2, t_prev1=0.0, t_prev2=0.0,
                            phi_tilde=U[dim * V:].copy())
    flags = rng.random(n) < 0.1
    mask = ConstraintMask(flags, np.zeros(n))
    params = MaterialParams(mu=1.3, lam=0.9, g_c=0.7, kappa=1e-10, eps=0.5, pressure_fn=lambda t: 10 * t)
    v = rng.standard_normal(n)
    ref = PhaseFieldOperator(disc.finest, st, mask, params, SplitKind.NOSPLIT).apply(v)
    info = lattice.info_from_mesh(fine)
    n_cells = [int(lattice.info_from_mesh(m).ncell[-1]) for m in levels]
    offs = info.plane_offsets()
    got = np.full(n, np.nan)
    for rank in range(world):
        part = D.SlabPartition(n_cells, world, rank, min_layers=2)
        L = n_levels - 1
        op = D.DistributedOperator(fine, L, part, st, mask, params, SplitKind.NOSPLIT)
        v_loc = torch.as_tensor(op.to_local(v), device="cuda")     # ghosts already true values
        out = torch.zeros(op.n_local, dtype=torch.float64, device="cuda")
        op.local.apply_dev(_lib.FULL, v_loc, out)
        # the overlapped form of DistributedOperator.apply_local: interior rows,
        # then the two boundary rows, must give the same owned values bitwise
        lo, hi = op.info.own if op.info.own != (0, 0) else (0, op.info.n_planes)
        if hi - lo >= 3:
            out2 = torch.zeros_like(out)
            op.local.apply_rows_dev(_lib.FULL, v_loc, out2, lo + 1, hi - 1)
            op.local.apply_rows_dev(_lib.FULL, v_loc, out2, lo, lo + 1)
            op.local.apply_rows_dev(_lib.FULL, v_loc, out2, hi - 1, hi)
            for sl in op.owned:
                assert torch.equal(out[sl], out2[sl])
            out3 = torch.zeros_like(out)
            op.local.apply_rows_dev(_lib.FULL, v_loc, out3, lo + 1, hi - 1)
            op.local.apply_ends_dev(_lib.FULL, v_loc, out3)                # PFFMG_HINT_ENDS
            for sl in op.owned:
                assert torch.equal(out[sl], out3[sl])
        s = part.slab(L)
        a, b = int(offs[s.own_lo]), int(offs[s.own_hi])
        per = b - a
        owned = torch.cat([out[sl] for sl in op.owned]).cpu().numpy()
        for c in range(dim + 1):
            got[c * V + a:c * V + b] = owned[c * per:(c + 1) * per]
    assert not np.isnan(got).any()
    assert rel_err(got, ref) <= 1e-14


@pytest.mark.parametrize("world", [2, 3])
def test_q2_slab_operator_stitches(world):
    """Q2 node-row slabs on the CUDA kernel: FULL vmult, both blocks, the
    diagonal and the semilinear residual of every rank's owned rows stitch to
    the whole-box result; the overlapped row split is bitwise identical."""
    from paper_1902_08112_b200 import _lib, distributed as D, lattice
    from paper_1902_08112_b200.fem import Discretization, build_q2_hierarchy
    from paper_1902_08112_b200.model import ConstraintMask, LinearizationState, MaterialParams, \
        PhaseFieldOperator, SplitKind
    disc = Discretization(build_q2_hierarchy(-2.0, 2.0, 4, 3))
    levels = disc.hierarchy.levels
    fine = levels[-1]
    V = fine.n_vertices
    n = 3 * V
    rng = np.random.default_rng(12)
    U = 1e-2 * rng.standard_normal(n)
    U[2 * V:] = np.clip(0.6 + 0.4 * rng.standard_normal(V), 0, 1)
    st = LinearizationState(U=U, U_prev1=U, U_prev2=U, t=0.2, t_prev1=0.0, t_prev2=0.0,
                            phi_tilde=U[2 * V:].copy())
    mask = ConstraintMask(rng.random(n) < 0.1, np.zeros(n))
    params = MaterialParams(mu=1.3, lam=0.9, g_c=0.7, kappa=1e-10, eps=0.5, pressure_fn=lambda t: 10 * t)
    v = rng.standard_normal(n)
    whole = PhaseFieldOperator(disc.finest, st, mask, params, SplitKind.NOSPLIT)
    vd = torch.as_tensor(v, device="cuda")
    refs = {}
    for which in (_lib.FULL, 0, 1):
        o = torch.zeros(n, dtype=torch.float64, device="cuda")
        if which == _lib.FULL:
            whole.apply_dev(which, vd, o)
        elif which == 0:
            whole.apply_dev(0, vd[:2 * V], o[:2 * V])
        else:
            whole.apply_dev(1, vd[2 * V:], o[2 * V:])
        refs[which] = o.cpu().numpy()
    d = torch.zeros(n, dtype=torch.float64, device="cuda")
    whole.diagonal_dev(d)
    refs["diag"] = d.cpu().numpy()
    r = torch.zeros(n, dtype=torch.float64, device="cuda")
    whole.semilinear_dev(r)
    refs["res"] = r.cpu().numpy()
    nxn = 2 * int(fine.ncell[0]) + 1
    got = {k: np.full(n, np.nan) for k in refs}
    L = len(levels) - 1
    for rank in range(world):
        part = D.SlabPartition([int(m.ncell[1]) for m in levels], world, rank, min_layers=2, order=2)
        op = D.DistributedOperator(fine, L, part, st, mask, params, SplitKind.NOSPLIT)
        Vl = op.info.n_vertices
        v_loc = torch.as_tensor(op.to_local(v), device="cuda")
        outs = {}
        for which in (_lib.FULL, 0, 1):
            o = torch.zeros(op.n_local, dtype=torch.float64, device="cuda")
            if which == _lib.FULL:
                op.local.apply_dev(which, v_loc, o)
            elif which == 0:
                op.local.apply_dev(0, v_loc[:2 * Vl], o[:2 * Vl])
            else:
                op.local.apply_dev(1, v_loc[2 * Vl:], o[2 * Vl:])
            outs[which] = o
        o = torch.zeros(op.n_local, dtype=torch.float64, device="cuda")
        op.local.diagonal_dev(o)
        outs["diag"] = o
        o = torch.zeros(op.n_local, dtype=torch.float64, device="cuda")
        op.local.semilinear_dev(o)
        outs["res"] = o
        lo, hi = op.info.own
        o2 = torch.zeros(op.n_local, dtype=torch.float64, device="cuda")
        op.local.apply_rows_dev(_lib.FULL, v_loc, o2, lo + 1, hi - 2)
        op.local.apply_rows_dev(_lib.FULL, v_loc, o2, lo, lo + 1)
        op.local.apply_rows_dev(_lib.FULL, v_loc, o2, hi - 2, hi)
        for sl in op.owned:
            assert torch.equal(outs[_lib.FULL][sl], o2[sl])
        s = part.slab(L)
        a, b = s.own_lo * nxn, s.own_hi * nxn
        per = b - a
        for k, o in outs.items():
            owned = torch.cat([o[sl] for sl in op.owned]).cpu().numpy()
            for c in range(3):
                got[k][c * V + a:c * V + b] = owned[c * per:(c + 1) * per]
    for k in refs:
        assert not np.isnan(got[k]).any(), k
        assert rel_err(got[k], refs[k]) <= 1e-14, k

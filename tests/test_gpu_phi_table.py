"""The per-QP a_phiphi table (pffmg_phi_coef, the phi-block entry of the
reference's _build_caches, model.py:270-309) against the on-the-fly
evaluation it replaces: the phi block, the block-diagonal smoother operator
and a Chebyshev step of it must agree to rounding on every lattice family
(2D/3D boxes, 2D/3D L-shapes, Q2), with and without a modulus field.  The
table is switched off per operator with PFFMG_PHI_TABLE=0 at construction."""
import os

import numpy as np
import pytest
import torch

from tests.golden.specs import MESHES
from tests.helpers import product_disc, product_params, product_state

pytestmark = pytest.mark.gpu

TOL = 1e-13


def _ops(space, U, pt, flags, params):
    from paper_1902_08112_b200 import model as M
    mask = M.ConstraintMask(flags, np.zeros(flags.size))
    st = product_state(U, pt, 0.1)
    tab = M.PhaseFieldOperator(space, st, mask, params, M.SplitKind.NOSPLIT)
    os.environ["PFFMG_PHI_TABLE"] = "0"
    try:
        fly = M.PhaseFieldOperator(space, st, mask, params, M.SplitKind.NOSPLIT)
    finally:
        del os.environ["PFFMG_PHI_TABLE"]
    assert tab._ptab is not None and fly._ptab is None
    return tab, fly


def _state(nc, V, seed):
    rng = np.random.default_rng(seed)
    U = 1e-3 * rng.standard_normal(nc * V)
    U[(nc - 1) * V:] = np.clip(0.7 + 0.3 * rng.standard_normal(V), 0.0, 1.0)
    pt = np.clip(U[(nc - 1) * V:] + 0.05 * rng.standard_normal(V), 0.0, 1.0)
    flags = rng.random(nc * V) < 0.1
    return U, pt, flags, rng


def _compare(tab, fly, rng):
    from paper_1902_08112_b200 import _lib
    n, d = tab.n_dofs, tab.dim * tab.V
    v = torch.as_tensor(rng.standard_normal(n), device="cuda")
    v[torch.as_tensor(np.asarray(tab.mask.is_constrained), device="cuda")] = 0.0   # pre-masked like the V-cycle
    for which, sl in ((_lib.BLOCKDIAG, slice(0, n)), (1, slice(d, n))):
        a, b = torch.empty_like(v[sl]), torch.empty_like(v[sl])
        tab.apply_dev(which, v[sl].contiguous(), a, pre=True)
        fly.apply_dev(which, v[sl].contiguous(), b, pre=True)
        torch.cuda.synchronize()
        err = float((a - b).norm() / b.norm())
        assert err <= TOL, (which, err)
    # one block-diagonal Chebyshev step (the smoother kernel of the V-cycle)
    r0 = torch.as_tensor(rng.standard_normal(n), device="cuda")
    x0 = torch.as_tensor(rng.standard_normal(n), device="cuda")
    inv = torch.as_tensor(1.0 + rng.random(n), device="cuda")
    cf = torch.tensor([0.3, 0.2], dtype=torch.float64, device="cuda")
    outs = []
    for op in (tab, fly):
        r, x, dn = r0.clone(), x0.clone(), torch.empty_like(v)
        op.cheb_step_bd(v, dn, r, x, inv, cf, cf, pre=True)
        torch.cuda.synchronize()
        outs.append((r, x, dn))
    for p, q in zip(*outs):
        assert float((p - q).norm() / q.norm()) <= TOL


@pytest.mark.parametrize("name", ["square", "lshape", "cfg1", "lshape3d", "lprism", "rect3d"])
@pytest.mark.parametrize("mod", [False, True])
def test_phi_table_matches_on_the_fly_q1(name, mod):
    disc = product_disc(name)
    space = disc.finest
    h = np.asarray(space.mesh.cell_size, float)
    if not np.all(h == h[0]):
        pytest.skip("anisotropic cells use the generic kernel (no table)")
    dim = MESHES[name][2]
    V = space.mesh.n_vertices
    U, pt, flags, rng = _state(dim + 1, V, 11)
    tab, fly = _ops(space, U, pt, flags, product_params(space, mod))
    _compare(tab, fly, rng)


@pytest.mark.parametrize("mod", [False, True])
def test_phi_table_matches_on_the_fly_q2(mod):
    from paper_1902_08112_b200.fem import Discretization, build_q2_hierarchy
    from paper_1902_08112_b200 import model as M
    from tests.golden.specs import modulus, params_for
    disc = Discretization(build_q2_hierarchy(0.0, 2.0, 2, 3))
    space = disc.finest
    V = space.mesh.n_vertices
    U, pt, flags, rng = _state(3, V, 5)
    params = params_for(space, modulus if mod else None, cls=M.MaterialParams)
    tab, fly = _ops(space, U, pt, flags, params)
    _compare(tab, fly, rng)

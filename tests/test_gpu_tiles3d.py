"""The 3D streaming kernels' work list (pffmg_lattice.tiles3d, ABI v3): the
occupied-tile list of a non-box lattice only changes which (tile, plane)
items the persistent grid distributes, never a result -- every mode is
bitwise the run over all tiles of the bounding lattice (NULL list), and the
list's tiles are exactly those holding a vertex."""
import ctypes

import numpy as np
import pytest
import torch

from tests.helpers import product_disc, product_params, product_state

pytestmark = pytest.mark.gpu


def _op(name, levels=None, seed=0):
    from paper_1902_08112_b200 import configs
    from paper_1902_08112_b200.model import ConstraintMask, PhaseFieldOperator, SplitKind
    rng = np.random.default_rng(seed)
    if name.startswith("cfg"):
        prob = configs.make(name, levels)
        space, st, params, n = prob.disc.finest, prob.state, prob.params, prob.n_dofs
    else:
        space = product_disc(name).finest
        V = space.mesh.n_vertices
        n = 4 * V
        U = 1e-3 * rng.standard_normal(n)
        U[3 * V:] = np.clip(0.7 + 0.3 * rng.standard_normal(V), 0.0, 1.0)
        pt = np.clip(U[3 * V:] + 0.05 * rng.standard_normal(V), 0.0, 1.0)
        st = product_state(U, pt, 0.1)
        params = product_params(space)
    flags = rng.random(n) < 0.1
    return PhaseFieldOperator(space, st, ConstraintMask(flags, np.zeros(n)), params, SplitKind.NOSPLIT), rng


def _runs(op, rng):
    from paper_1902_08112_b200 import _lib
    n, d = op.n_dofs, op.dim * op.V
    v = torch.as_tensor(rng.standard_normal(n), device="cuda")
    outs = []
    for which, sl in ((_lib.FULL, slice(0, n)), (0, slice(0, d)), (1, slice(d, n)), (_lib.BLOCKDIAG, slice(0, n))):
        o = torch.empty_like(v[sl])
        op.apply_dev(which, v[sl].contiguous(), o)
        outs.append(o)
    r = torch.empty_like(v)
    op.residual_dev(_lib.FULL, v, v, r)
    outs.append(r)
    return outs


@pytest.mark.parametrize("name,levels", [("lprism", None), ("lshape3d", None), ("cfg4", 4)])
def test_tile_list_is_bitwise_all_tiles(name, levels):
    from paper_1902_08112_b200 import lattice
    op, rng = _op(name, levels)
    L = op.lat.struct
    assert L.tiles3d, "a non-box 3D lattice carries its occupied-tile list"
    # the list: exactly the TILE3 x TILE3 column tiles that hold a vertex
    info = op.lat.info
    occ = np.zeros((int(info.ncell[1]) + 1, int(info.ncell[0]) + 1), bool)
    _, vlo, vhi, _, _ = info.rows
    vlo = np.asarray(vlo).reshape(-1, occ.shape[0])
    vhi = np.asarray(vhi).reshape(-1, occ.shape[0])
    for z in range(vlo.shape[0]):
        for y in range(occ.shape[0]):
            occ[y, vlo[z, y]:vhi[z, y]] = True
    T = lattice.TILE3
    ntx = -(-occ.shape[1] // T)
    want = sorted({(y // T) * ntx + x // T for y, x in zip(*np.nonzero(occ))})
    assert list(lattice.occupied_tiles3d(info)) == want
    state = rng.bit_generator.state
    with_list = _runs(op, rng)
    saved = (L.tiles3d, L.n_tiles3d)
    L.tiles3d, L.n_tiles3d = None, 0
    try:
        rng.bit_generator.state = state
        without = _runs(op, rng)
    finally:
        L.tiles3d, L.n_tiles3d = saved
    for a, b in zip(with_list, without):
        assert torch.equal(a, b)

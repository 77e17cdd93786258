"""GPU quantities of interest (libpffmg pffmg_qoi) vs the reference's values
(model.py:472-504): crack energy, bulk energy (both splits, blended Miehe,
modulus field, pressure work) and fracture volume, <= 1e-12 relative."""
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from tests.golden.specs import MESHES
from tests.helpers import product_disc, product_params, product_state

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.mark.parametrize("name", list(MESHES))
def test_qoi_match_reference(golden, name):
    from paper_1902_08112_b200 import model as M
    g = golden["qoi"]
    space = product_disc(name).finest
    U = g[f"{name}/U"]
    V = space.mesh.n_vertices if hasattr(space.mesh, "n_vertices") else U.size // (space.mesh.dim + 1)
    st = product_state(U, U[-V:], g[f"{name}/t"])
    for variant in ("plain", "modulus"):
        params = product_params(space, variant == "modulus")

        def close(a, key):
            ref = float(g[key])
            assert abs(a - ref) <= TOL * abs(ref), (key, a, ref)
        close(M.crack_energy(space, st, params), f"{name}/{variant}/crack_energy")
        close(M.fracture_volume(space, U), f"{name}/{variant}/fracture_volume")
        close(M.fracture_volume(space, torch.as_tensor(U, device="cuda")), f"{name}/{variant}/fracture_volume")
        for split, sk in (("none", M.SplitKind.NOSPLIT), ("miehe", M.SplitKind.MIEHE)):
            close(M.bulk_energy(space, st, params, sk), f"{name}/{variant}/{split}/bulk_energy")
        params.split_band = 0.05
        close(M.bulk_energy(space, st, params, M.SplitKind.MIEHE), f"{name}/{variant}/miehe_band/bulk_energy")


def test_qoi_deterministic():
    from paper_1902_08112_b200 import configs
    from paper_1902_08112_b200 import model as M
    prob = configs.make("cfg1")
    a = [M.bulk_energy(prob.disc.finest, prob.state, prob.params, M.SplitKind.MIEHE) for _ in range(3)]
    assert a[0] == a[1] == a[2]
    assert np.isfinite(a[0])


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("variant", ["plain", "modulus"])
@pytest.mark.parametrize("key", ["none", "miehe", "miehe_band"])
def test_boundary_load_matches_reference(golden, name, variant, key):
    """boundary_load (model.py:511-547) for every tag and direction, on the
    lattice-native mesh and on the reference-shaped (keys/cells) mesh."""
    from paper_1902_08112_b200 import model as M
    from paper_1902_08112_b200.fem import build_hierarchy
    from tests.golden.specs import face_tagger
    g = golden["boundary"]
    blocks, n_levels, dim = MESHES[name]
    mesh = build_hierarchy(blocks, n_levels, dim, face_tagger).finest
    space = SimpleNamespace(mesh=mesh, dim=dim)
    params = product_params(space, variant == "modulus")
    params.split_band = 0.05 if key == "miehe_band" else 0.0
    split = M.SplitKind.NOSPLIT if key == "none" else M.SplitKind.MIEHE
    st = product_state(g[f"{name}/U"], None, 0.1)
    ref = g[f"{name}/{variant}/{key}/load"]
    scale = np.abs(ref).max()
    got = np.array([[M.boundary_load(space, st, params, split, tag, d) for d in range(dim)]
                    for tag in range(4)])
    assert np.all(np.abs(got - ref) <= 1e-12 * scale), (got, ref)
    # the same through a reference-shaped mesh object (arrays only, as patch.install feeds it)
    ref_mesh = SimpleNamespace(keys=mesh.keys, cells=mesh.cells, cell_size=mesh.cell_size,
                               vertices=mesh.vertices, bf_cell=mesh.bf_cell, bf_face=mesh.bf_face,
                               bf_tag=mesh.bf_tag, dim=dim, n_vertices=mesh.n_vertices)
    space2 = SimpleNamespace(mesh=ref_mesh, dim=dim)
    got2 = np.array([[M.boundary_load(space2, st, params, split, tag, d) for d in range(dim)]
                     for tag in range(4)])
    assert np.all(np.abs(got2 - ref) <= 1e-12 * scale)
    with pytest.raises(ValueError):
        M.boundary_load(space, st, params, split, 7, 0)

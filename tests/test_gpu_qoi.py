"""GPU quantities of interest (libpffmg pffmg_qoi) vs the reference's values
(model.py:472-504): crack energy, bulk energy (both splits, blended Miehe,
modulus field, pressure work) and fracture volume, <= 1e-12 relative."""
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

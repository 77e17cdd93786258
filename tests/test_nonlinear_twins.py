"""Active-set helpers vs the reference's outputs
(tests/golden/make_golden_nonlinear.py).  The set must be bit-exact."""
import numpy as np
import pytest

from tests.conftest import Golden
from tests.helpers import product_disc

NAMES = ["square", "lshape3d", "cfg1"]


@pytest.mark.parametrize("name", NAMES)
def test_lumped_mass_inverse_matches_reference(name):
    from paper_1902_08112_b200.nonlinear import lumped_mass_inverse
    g = Golden("nonlinear")
    disc = product_disc(name)
    assert np.array_equal(lumped_mass_inverse(disc.finest), g[f"{name}/mass_inv"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_active_set_bit_exact(name):
    from paper_1902_08112_b200.nonlinear import compute_active_set

    class P:
        c = 100.0

    g = Golden("nonlinear")
    disc = product_disc(name)
    dm = disc.finest.dofmap
    for k in range(3):
        got = compute_active_set(g[f"{name}/{k}/R"], g[f"{name}/{k}/U"], g[f"{name}/{k}/phi_old"],
                                 g[f"{name}/mass_inv"], P, dm,
                                 dirichlet_flags=g[f"{name}/{k}/dflags"] if k == 2 else None)
        assert got.dtype == bool
        assert np.array_equal(got, g[f"{name}/{k}/active"])

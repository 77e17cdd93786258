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


def test_lanczos_batch_equals_one_by_one():
    """Batched spectrum extraction (the setup's one host step) is bit-identical
    to the per-run lanczos_extremes (krylov.py:187-198), fallbacks included."""
    from paper_1902_08112_b200.krylov import CG_MAXIT, lanczos_extremes, lanczos_extremes_batch
    rng = np.random.default_rng(7)
    rows = []
    for k in (10, 10, 7, 1, 10, 3, 0, 2, 10):
        r = np.zeros(8 + 2 * CG_MAXIT)
        r[4], r[5] = k, max(k - 1, 0)
        r[8:8 + k] = rng.uniform(0.1, 2.0, k)
        r[8 + CG_MAXIT:8 + CG_MAXIT + max(k - 1, 0)] = rng.uniform(0.01, 1.0, max(k - 1, 0))
        rows.append(r)
    one = [lanczos_extremes(r, 10) for r in rows]
    batch = lanczos_extremes_batch(np.array(rows), 10)
    for a, b in zip(one, batch):
        assert (a.lambda_min_hat, a.lambda_max_hat, a.fallback) == (b.lambda_min_hat, b.lambda_max_hat, b.fallback)

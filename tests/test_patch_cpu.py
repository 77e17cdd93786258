"""The drop-in installer swaps module attributes of the reference (CPU only;
skipped where the reference is not importable, e.g. on the GPU box)."""
import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture
def fracmg():
    if not os.path.isdir(REF):
        pytest.skip("reference not available here")
    sys.path.insert(0, REF)
    import fracmg  # noqa: F401
    yield sys.modules["fracmg"]
    sys.path.remove(REF)


def test_install_and_uninstall(fracmg):
    from paper_1902_08112_b200 import krylov, mgsolve, patch
    orig = fracmg.mgsolve.vcycle
    patch.install(fracmg)
    try:
        assert fracmg.mgsolve.vcycle is mgsolve.vcycle
        assert fracmg.mgsolve.build_level_contexts is mgsolve.build_level_contexts
        assert fracmg.krylov.gmres is krylov.gmres
        assert krylov._NO_CONVERGENCE[0] is fracmg.krylov.NoConvergence
    finally:
        patch.uninstall()
    assert fracmg.mgsolve.vcycle is orig
    assert krylov._NO_CONVERGENCE[0] is krylov.NoConvergence


def test_install_physics(fracmg):
    from paper_1902_08112_b200 import model, nonlinear, patch
    orig = fracmg.model.residual
    patch.install(fracmg, operator=True, physics=True)
    try:
        assert fracmg.model.residual is model.residual
        assert fracmg.model.bulk_energy is model.bulk_energy
        assert fracmg.model.PhaseFieldOperator is model.PhaseFieldOperator
        assert fracmg.nonlinear.compute_active_set is nonlinear.compute_active_set
    finally:
        patch.uninstall()
    assert fracmg.model.residual is orig

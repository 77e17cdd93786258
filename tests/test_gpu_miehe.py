"""CUDA Miehe spectral split (2D and 3D) vs the reference's golden outputs and the
CPU oracle (model.py:56-86 blend, 148-219 _split_batch, 270-413 operator,
420-460 residual).  Bar: <= 1e-12 relative 2-norm error, as for NoSplit."""
import numpy as np
import pytest
import torch

from oracle import jacobian
from tests.conftest import rel_err
from tests.golden.specs import MESHES
from tests.helpers import (oracle_material, oracle_state, product_disc, product_params,
                           product_state)

pytestmark = pytest.mark.gpu

TOL = 1e-12
MESH2D = [m for m, spec in MESHES.items() if spec[2] == 2]
MESH3D = [m for m, spec in MESHES.items() if spec[2] == 3]
CASES = [(m, f, v) for m in MESHES for f in ("operator", "operator_band") for v in ("plain", "masked")]


def _case(golden, name, fixture, variant):
    from paper_1902_08112_b200 import model as M
    g = golden[fixture]
    tag = f"{name}/{'miehe' if fixture == 'operator' else 'miehe_band'}/{variant}"
    space = product_disc(name).finest
    st = product_state(g[f"{tag}/U"], g[f"{tag}/phi_tilde"], g[f"{tag}/t"])
    flags = g[f"{tag}/flags"]
    mask = M.ConstraintMask(flags, np.zeros(flags.size))
    params = product_params(space)
    params.split_band = float(g[f"{tag}/band"]) if g.has(f"{tag}/band") else 0.0
    return g, tag, space, st, mask, params


@pytest.mark.parametrize("name,fixture,variant", CASES)
def test_miehe_operator_matches_reference(golden, name, fixture, variant):
    from paper_1902_08112_b200 import model as M
    g, tag, space, st, mask, params = _case(golden, name, fixture, variant)
    op = M.PhaseFieldOperator(space, st, mask, params, M.SplitKind.MIEHE)
    v = g[f"{tag}/v"]
    d = op.dim * op.V
    out = op.apply(v)
    assert rel_err(out, g[f"{tag}/apply"]) <= TOL
    assert rel_err(op.apply_block(0, v[:d]), g[f"{tag}/apply_u"]) <= TOL
    assert rel_err(op.apply_block(1, v[d:]), g[f"{tag}/apply_phi"]) <= TOL
    diag = op.diagonal()
    assert rel_err(diag, g[f"{tag}/diagonal"]) <= TOL
    flags = g[f"{tag}/flags"]
    assert np.array_equal(out[flags], v[flags])
    assert np.all(diag[flags] == 1.0)
    res = M.residual(space, st, mask, params, M.SplitKind.MIEHE)
    assert rel_err(res, g[f"{tag}/residual"]) <= TOL
    assert np.all(res[flags] == 0.0)


@pytest.mark.parametrize("name", list(MESHES))
def test_miehe_premasked_and_deterministic(golden, name):
    from paper_1902_08112_b200 import _lib
    from paper_1902_08112_b200 import model as M
    g, tag, space, st, mask, params = _case(golden, name, "operator_band", "masked")
    op = M.PhaseFieldOperator(space, st, mask, params, M.SplitKind.MIEHE)
    flags = torch.as_tensor(g[f"{tag}/flags"], device="cuda")
    v = torch.as_tensor(g[f"{tag}/v"], device="cuda").clone()
    v[flags] = 0.0
    d = op.dim * op.V
    for which, vin, n in ((_lib.FULL, v, op.n_dofs), (0, v[:d], d), (1, v[d:], op.V)):
        a = torch.empty(n, dtype=torch.float64, device="cuda")
        b = torch.empty_like(a)
        c = torch.empty_like(a)
        op.apply_dev(which, vin, a)
        op.apply_dev(which, vin, b, pre=True)
        op.apply_dev(which, vin, c)
        assert torch.equal(a, b) and torch.equal(a, c)


@pytest.mark.parametrize("band", [0.0, 0.02])
def test_miehe_larger_states_vs_oracle(band):
    """A refinement beyond the golden files, with a modulus field (no golden
    case carries one for Miehe): CUDA vs the oracle directly."""
    from paper_1902_08112_b200.fem import Discretization, build_hierarchy
    from paper_1902_08112_b200.model import ConstraintMask, PhaseFieldOperator, SplitKind
    from oracle import fe, meshgen
    from tests.golden.specs import modulus
    blocks, n_levels, dim = MESHES["lshape"]
    n_levels += 1
    olev = meshgen.build_hierarchy(blocks, n_levels, dim)[-1]
    T = fe.LevelTables(olev, n_levels - 1)
    rng = np.random.default_rng(31)
    n = T.n_dofs
    h = float(np.min(olev.cell_size))
    U = 0.1 * h * rng.standard_normal(n)
    U[T.phi_slice] = np.clip(0.6 + 0.4 * rng.standard_normal(T.n_vertices), 0, 1)
    pt = np.clip(U[T.phi_slice] + 0.05 * rng.standard_normal(T.n_vertices), 0, 1)
    flags = rng.random(n) < 0.1
    v = rng.standard_normal(n)
    mat = oracle_material(T, True)
    mat.split_band = band
    ref_op = jacobian.JacobianOperator(T, oracle_state(U, pt, 0.3), flags, mat, "miehe")
    space = Discretization(build_hierarchy(blocks, n_levels, dim)).finest
    params = product_params(space, True)
    params.split_band = band
    st = product_state(U, pt, 0.3)
    mask = ConstraintMask(flags, np.zeros(n))
    op = PhaseFieldOperator(space, st, mask, params, SplitKind.MIEHE)
    d = T.dim * T.n_vertices
    assert rel_err(op.apply(v), ref_op.apply(v)) <= TOL
    assert rel_err(op.apply_block(0, v[:d]), ref_op.apply_block(0, v[:d])) <= TOL
    assert rel_err(op.apply_block(1, v[d:]), ref_op.apply_block(1, v[d:])) <= TOL
    assert rel_err(op.diagonal(), ref_op.diagonal()) <= TOL
    from paper_1902_08112_b200 import model as M
    res = M.residual(space, st, mask, params, SplitKind.MIEHE)
    assert rel_err(res, jacobian.residual(T, oracle_state(U, pt, 0.3), flags, mat, "miehe")) <= TOL


@pytest.mark.parametrize("name", ["lprism", "rect3d"])
def test_miehe3d_larger_states_vs_oracle(name):
    """3D refinement beyond the golden files (incl. anisotropic cells) with a
    modulus field and the blend: CUDA vs the oracle directly."""
    from paper_1902_08112_b200.fem import Discretization, build_hierarchy
    from paper_1902_08112_b200.model import ConstraintMask, PhaseFieldOperator, SplitKind
    from paper_1902_08112_b200 import model as M
    from oracle import fe, meshgen
    blocks, n_levels, dim = MESHES[name]
    n_levels += 1
    olev = meshgen.build_hierarchy(blocks, n_levels, dim)[-1]
    T = fe.LevelTables(olev, n_levels - 1)
    rng = np.random.default_rng(32)
    n = T.n_dofs
    h = float(np.min(olev.cell_size))
    U = 0.1 * h * rng.standard_normal(n)
    U[T.phi_slice] = np.clip(0.6 + 0.4 * rng.standard_normal(T.n_vertices), 0, 1)
    pt = np.clip(U[T.phi_slice] + 0.05 * rng.standard_normal(T.n_vertices), 0, 1)
    flags = rng.random(n) < 0.1
    v = rng.standard_normal(n)
    mat = oracle_material(T, True)
    mat.split_band = 0.03
    ref_op = jacobian.JacobianOperator(T, oracle_state(U, pt, 0.3), flags, mat, "miehe")
    space = Discretization(build_hierarchy(blocks, n_levels, dim)).finest
    params = product_params(space, True)
    params.split_band = 0.03
    st = product_state(U, pt, 0.3)
    mask = ConstraintMask(flags, np.zeros(n))
    op = PhaseFieldOperator(space, st, mask, params, SplitKind.MIEHE)
    d = T.dim * T.n_vertices
    assert rel_err(op.apply(v), ref_op.apply(v)) <= TOL
    assert rel_err(op.apply_block(0, v[:d]), ref_op.apply_block(0, v[:d])) <= TOL
    assert rel_err(op.apply_block(1, v[d:]), ref_op.apply_block(1, v[d:])) <= TOL
    assert rel_err(op.diagonal(), ref_op.diagonal()) <= TOL
    res = M.residual(space, st, mask, params, SplitKind.MIEHE)
    assert rel_err(res, jacobian.residual(T, oracle_state(U, pt, 0.3), flags, mat, "miehe")) <= TOL

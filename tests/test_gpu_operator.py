"""CUDA operator (libpffmg via the PhaseFieldOperator twin) vs the reference's
golden outputs and vs the CPU oracle.  Bar: <= 1e-12 relative 2-norm error
(north_star), constrained rows bit-equal to the input, constrained diagonal
entries exactly 1.0, bitwise reproducible runs."""
import numpy as np
import pytest
import torch

from oracle import jacobian
from tests.conftest import rel_err
from tests.golden.specs import MESHES
from tests.helpers import (OP_TAGS, oracle_material, oracle_stack, oracle_state, product_disc,
                           product_params, product_state)

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _op(g, name, variant, split="none"):
    from paper_1902_08112_b200.model import ConstraintMask, PhaseFieldOperator, SplitKind
    tag = f"{name}/{split}/{variant}"
    disc = product_disc(name)
    space = disc.finest
    st = product_state(g[f"{tag}/U"], g[f"{tag}/phi_tilde"], g[f"{tag}/t"])
    flags = g[f"{tag}/flags"]
    mask = ConstraintMask(flags, np.zeros(flags.size))
    op = PhaseFieldOperator(space, st, mask, product_params(space, variant == "modulus"),
                            SplitKind.NOSPLIT)
    return op, tag


@pytest.mark.parametrize("name,variant", OP_TAGS)
def test_apply_matches_reference(golden, name, variant):
    g = golden["operator"]
    op, tag = _op(g, name, variant)
    v = g[f"{tag}/v"]
    d = op.dim * op.V
    out = op.apply(v)
    assert isinstance(out, np.ndarray)
    assert rel_err(out, g[f"{tag}/apply"]) <= TOL
    assert rel_err(op.apply_block(0, v[:d]), g[f"{tag}/apply_u"]) <= TOL
    assert rel_err(op.apply_block(1, v[d:]), g[f"{tag}/apply_phi"]) <= TOL
    diag = op.diagonal()
    assert rel_err(diag, g[f"{tag}/diagonal"]) <= TOL
    flags = g[f"{tag}/flags"]
    assert np.array_equal(out[flags], v[flags])           # identity rows, bit-exact
    assert np.all(diag[flags] == 1.0)


@pytest.mark.parametrize("name", list(MESHES))
def test_tensor_io_zero_copy_and_deterministic(golden, name):
    g = golden["operator"]
    op, tag = _op(g, name, "masked")
    v = torch.as_tensor(g[f"{tag}/v"], device="cuda")
    a = op.apply(v)
    b = op.apply(v)
    assert a.is_cuda and torch.equal(a, b)                # bitwise reproducible
    assert rel_err(a.cpu().numpy(), g[f"{tag}/apply"]) <= TOL


@pytest.mark.parametrize("name", ["cfg1", "lshape3d", "cube"])
def test_zero_vector_and_linearity(golden, name):
    g = golden["operator"]
    op, tag = _op(g, name, "masked")
    n = op.n_dofs
    assert not op.apply(np.zeros(n)).any()
    rng = np.random.default_rng(3)
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    lhs = op.apply(x + 0.37 * y)
    rhs = op.apply(x) + 0.37 * op.apply(y)
    assert rel_err(lhs, rhs) <= 1e-13


@pytest.mark.parametrize("name", ["cfg1", "lprism"])
def test_block_structure_matches_full(golden, name):
    """apply_block == restriction of apply to the block, coupling G_u_phi = 0
    (reference tests/test_model.py:229-276)."""
    g = golden["operator"]
    op, tag = _op(g, name, "masked")
    n, d = op.n_dofs, op.dim * op.V
    rng = np.random.default_rng(4)
    vu = rng.standard_normal(d)
    full = op.apply(np.concatenate([vu, np.zeros(n - d)]))
    assert rel_err(full[:d], op.apply_block(0, vu)) <= 1e-14
    vp = rng.standard_normal(n - d)
    full = op.apply(np.concatenate([np.zeros(d), vp]))
    flags = g[f"{tag}/flags"]
    assert np.all(full[:d][~flags[:d]] == 0.0)            # G_u_phi = 0 exactly
    assert rel_err(full[d:], op.apply_block(1, vp)) <= 1e-14


@pytest.mark.parametrize("name", ["rect3d", "lprism", "cfg1"])
def test_larger_random_states_vs_oracle(name):
    """Finer refinement than the golden files: compare with the oracle directly."""
    from paper_1902_08112_b200.fem import Discretization, build_hierarchy
    from paper_1902_08112_b200.model import ConstraintMask, PhaseFieldOperator, SplitKind
    from oracle import fe, meshgen
    blocks, n_levels, dim = MESHES[name]
    n_levels += 1
    olev = meshgen.build_hierarchy(blocks, n_levels, dim)[-1]
    T = fe.LevelTables(olev, n_levels - 1)
    rng = np.random.default_rng(8)
    n = T.n_dofs
    U = 1e-2 * rng.standard_normal(n)
    U[T.phi_slice] = np.clip(0.6 + 0.4 * rng.standard_normal(T.n_vertices), 0, 1)
    pt = np.clip(U[T.phi_slice] + 0.05 * rng.standard_normal(T.n_vertices), 0, 1)
    flags = rng.random(n) < 0.1
    v = rng.standard_normal(n)
    mat = oracle_material(T)
    ref_op = jacobian.JacobianOperator(T, oracle_state(U, pt, 0.3), flags, mat)
    disc = Discretization(build_hierarchy(blocks, n_levels, dim))
    space = disc.finest
    op = PhaseFieldOperator(space, product_state(U, pt, 0.3), ConstraintMask(flags, np.zeros(n)),
                            product_params(space), SplitKind.NOSPLIT)
    assert rel_err(op.apply(v), ref_op.apply(v)) <= TOL
    d = T.dim * T.n_vertices
    assert rel_err(op.apply_block(0, v[:d]), ref_op.apply_block(0, v[:d])) <= TOL
    assert rel_err(op.apply_block(1, v[d:]), ref_op.apply_block(1, v[d:])) <= TOL
    assert rel_err(op.diagonal(), ref_op.diagonal()) <= TOL


@pytest.mark.parametrize("name", ["cfg1", "lshape", "lprism", "cube"])
def test_premasked_hint_is_exact(golden, name):
    """PFFMG_HINT_PREMASKED (used inside the V-cycle / CG) gives bit-identical
    results when the input is zero at constrained dofs."""
    from paper_1902_08112_b200 import _lib
    g = golden["operator"]
    op, tag = _op(g, name, "masked")
    flags = torch.as_tensor(g[f"{tag}/flags"], device="cuda")
    v = torch.as_tensor(g[f"{tag}/v"], device="cuda").clone()
    v[flags] = 0.0
    d = op.dim * op.V
    for which, vin, n in ((_lib.FULL, v, op.n_dofs), (0, v[:d], d), (1, v[d:], op.V)):
        a, b = torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64, device="cuda")
        op.apply_dev(which, vin, a)
        op.apply_dev(which, vin, b, pre=True)
        assert torch.equal(a, b)


def test_fused_epilogues_match_unfused(golden):
    """residual / Chebyshev epilogues == separate apply + vector algebra."""
    from paper_1902_08112_b200 import _lib
    g = golden["operator"]
    op, tag = _op(g, "cfg1", "masked")
    n, d = op.n_dofs, op.dim * op.V
    rng = np.random.default_rng(5)
    dev = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
    x, b = dev(rng.standard_normal(n)), dev(rng.standard_normal(n))
    out = torch.empty_like(x)
    op.residual_dev(_lib.FULL, x, b, out)
    assert rel_err(out.cpu().numpy(), (b - op.apply(x)).cpu().numpy()) <= 1e-14
    # Chebyshev step on the u block
    din = dev(rng.standard_normal(d))
    r0 = dev(rng.standard_normal(d))
    x0 = dev(rng.standard_normal(d))
    inv = dev(1.0 / (1.0 + rng.random(d)))
    r, xx, dout = r0.clone(), x0.clone(), torch.empty_like(din)
    op.cheb_step_dev(0, din, dout, r, xx, inv, 0.3, 0.7)
    r_ref = r0 - op.apply_block(0, din)
    d_ref = 0.3 * din + 0.7 * (inv * r_ref)
    assert torch.equal(r, r_ref)
    assert rel_err(dout.cpu().numpy(), d_ref.cpu().numpy()) <= 1e-15
    assert rel_err(xx.cpu().numpy(), (x0 + d_ref).cpu().numpy()) <= 1e-15


@pytest.mark.parametrize("name,variant", OP_TAGS)
def test_semilinear_residual_matches_reference(golden, name, variant):
    """model.residual twin (NoSplit) vs the reference's A(U) (model.py:420-460)."""
    from paper_1902_08112_b200 import model as M
    g = golden["operator"]
    tag = f"{name}/none/{variant}"
    disc = product_disc(name)
    space = disc.finest
    st = product_state(g[f"{tag}/U"], g[f"{tag}/phi_tilde"], g[f"{tag}/t"])
    flags = g[f"{tag}/flags"]
    mask = M.ConstraintMask(flags, np.zeros(flags.size))
    out = M.residual(space, st, mask, product_params(space, variant == "modulus"), M.SplitKind.NOSPLIT)
    assert isinstance(out, np.ndarray)
    assert rel_err(out, g[f"{tag}/residual"]) <= TOL
    assert np.all(out[flags] == 0.0)


@pytest.mark.parametrize("name", ["cfg1", "lshape", "lprism", "cube"])
def test_pinned_host_apply_pipeline_is_exact(golden, name):
    """pffmg_apply_host (H2D / stencil / D2H overlapped by plane strips) gives
    bit-identical results to the device apply for any strip count."""
    import ctypes
    from paper_1902_08112_b200 import _lib
    g = golden["operator"]
    op, tag = _op(g, name, "masked")
    v = torch.as_tensor(g[f"{tag}/v"]).pin_memory()
    ref = op.apply(v.cuda()).cpu()
    assert torch.equal(op.apply(v), ref)                          # public path
    out = torch.empty_like(v).pin_memory()
    assert op.apply(v, out=out) is out and torch.equal(out, ref)
    d_in, d_out = torch.empty_like(ref).cuda(), torch.empty_like(ref).cuda()
    po = op.lat.plane_off_host
    for strips in (1, 2, 3, 7, 64):
        out.zero_()
        _lib.call("pffmg_apply_host", op.lat.ref, op._stp, _lib.FULL, ctypes.c_void_p(v.data_ptr()),
                  ctypes.c_void_p(out.data_ptr()), _lib.ptr(d_in), _lib.ptr(d_out),
                  None if po is None else po.ctypes.data, strips, _lib.stream())
        torch.cuda.synchronize()
        assert torch.equal(out, ref), strips


@pytest.mark.parametrize("name", ["cfg1", "lshape", "lprism", "cube"])
def test_pageable_host_apply_pipeline_is_exact(golden, name, monkeypatch):
    """pffmg_apply_pageable (numpy in / out: threaded staging through page-locked
    buffers, pipelined with the copies and the stencil) gives bit-identical
    results to the device apply for any strip count; PhaseFieldOperator.apply
    takes it for numpy vectors above PAGEABLE_MIN dofs."""
    from paper_1902_08112_b200 import _lib, model
    g = golden["operator"]
    op, tag = _op(g, name, "masked")
    v = np.ascontiguousarray(g[f"{tag}/v"], dtype=np.float64)
    ref = op.apply(torch.as_tensor(v).cuda()).cpu().numpy()
    calls = []
    real = _lib.call
    monkeypatch.setattr(_lib, "call", lambda name_, *a: (calls.append(name_), real(name_, *a))[1])
    monkeypatch.setattr(model, "PAGEABLE_MIN", 1)
    got = op.apply(v)                                             # public path, numpy -> numpy
    assert "pffmg_apply_pageable" in calls
    assert isinstance(got, np.ndarray) and np.array_equal(got, ref)
    out = np.full_like(v, np.nan)
    assert op.apply(v, out=out) is out and np.array_equal(out, ref)
    monkeypatch.setattr(model, "PAGEABLE_PIPELINE", False)        # plain copies: same values
    calls.clear()
    assert np.array_equal(op.apply(v), ref) and "pffmg_apply_pageable" not in calls
    d_in, d_out = torch.empty(v.size, dtype=torch.float64, device="cuda"), torch.empty(v.size, dtype=torch.float64,
                                                                                      device="cuda")
    po = op.lat.plane_off_host
    for strips in (1, 2, 3, 7, 64):
        out[:] = np.nan
        real("pffmg_apply_pageable", op.lat.ref, op._stp, _lib.FULL, v.ctypes.data, out.ctypes.data,
             _lib.ptr(d_in), _lib.ptr(d_out), None if po is None else po.ctypes.data, strips, _lib.stream())
        assert np.array_equal(out, ref), strips


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("split", ["none", "miehe"])
def test_blockdiag_operator_equals_blocks(golden, name, split):
    """PFFMG_BLOCKDIAG (both diagonal blocks in one kernel, the block smoother's
    operator) == [apply_block(0); apply_block(1)]."""
    from paper_1902_08112_b200 import _lib
    from paper_1902_08112_b200.model import ConstraintMask, PhaseFieldOperator, SplitKind
    g = golden["operator"]
    tag = f"{name}/{split}/masked"
    space = product_disc(name).finest
    st = product_state(g[f"{tag}/U"], g[f"{tag}/phi_tilde"], g[f"{tag}/t"])
    flags = g[f"{tag}/flags"]
    op = PhaseFieldOperator(space, st, ConstraintMask(flags, np.zeros(flags.size)), product_params(space),
                            SplitKind.MIEHE if split == "miehe" else SplitKind.NOSPLIT)
    v = torch.as_tensor(g[f"{tag}/v"], device="cuda")
    d = op.dim * op.V
    out = torch.empty_like(v)
    op.apply_dev(_lib.BLOCKDIAG, v, out)
    ref = torch.cat([op.apply_block(0, v[:d]), op.apply_block(1, v[d:])])
    assert rel_err(out.cpu().numpy(), ref.cpu().numpy()) <= 1e-14
    assert rel_err(out[:d].cpu().numpy(), ref[:d].cpu().numpy()) <= 1e-14
    assert rel_err(out[d:].cpu().numpy(), ref[d:].cpu().numpy()) <= 1e-14


@pytest.mark.parametrize("name,variant", [t for t in OP_TAGS if MESHES[t[0]][2] == 3])
def test_phi_block_table_matches_recomputed(golden, name, variant, monkeypatch):
    """3D isotropic levels cache a_phiphi per QP (pffmg_phi_coef, the reference's
    _build_caches entry model.py:304-308): the phi block, its Chebyshev step
    and residual read the table; they must agree with the path that re-derives
    a_phiphi from U (PFFMG_PHI_TABLE=0) and with the reference golden."""
    from paper_1902_08112_b200 import _lib
    g = golden["operator"]
    op, tag = _op(g, name, variant)
    if not np.all(np.asarray(op.lat.info.h) == op.lat.info.h[0]):
        pytest.skip("anisotropic cells: generic kernel, no table")
    assert op._ptab is not None and op._st.phi_coef == op._ptab.data_ptr()
    monkeypatch.setenv("PFFMG_PHI_TABLE", "0")
    op0, _ = _op(g, name, variant)
    assert op0._ptab is None
    d = op.dim * op.V
    v = torch.as_tensor(g[f"{tag}/v"][d:], device="cuda")
    a, b = torch.empty_like(v), torch.empty_like(v)
    op.apply_dev(1, v, a)
    op0.apply_dev(1, v, b)
    assert rel_err(a.cpu().numpy(), b.cpu().numpy()) <= 1e-13
    assert rel_err(a.cpu().numpy(), g[f"{tag}/apply_phi"]) <= TOL
    r0 = torch.randn_like(v)
    x0 = torch.randn_like(v)
    inv = torch.rand_like(v) + 1.0
    outs = []
    for o in (op, op0):
        r, x, dd = r0.clone(), x0.clone(), torch.empty_like(v)
        o.cheb_step_dev(1, v, dd, r, x, inv, 0.3, 0.2)
        outs.append((r, x, dd))
    for p, q in zip(*outs):
        assert (p - q).norm() <= 1e-13 * q.norm()

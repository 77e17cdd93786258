"""Property tests mirroring the reference's own: finite-difference
Jacobian of the GPU residual vs the GPU operator (tests/test_model.py:211-226),
V-cycle zero / linearity / constrained neutrality (tests/test_mgsolve.py:
186-255), GMRES h-robustness over refinements (tests/test_mgsolve.py:342-363),
and edge cases: all-constrained masks, one-cell meshes, one-level
hierarchies."""
import numpy as np
import pytest
import torch

from tests.conftest import rel_err
from tests.golden.specs import MESHES, params_for

pytestmark = pytest.mark.gpu


def _space(name, extra=0):
    from paper_1902_08112_b200.fem import Discretization, build_hierarchy
    blocks, n_levels, dim = MESHES[name]
    return Discretization(build_hierarchy(blocks, n_levels + extra, dim))


def _state(space, seed, scale=1e-2):
    from paper_1902_08112_b200.model import LinearizationState
    rng = np.random.default_rng(seed)
    V = space.mesh.n_vertices
    dim = space.mesh.dim
    h = float(np.min(space.mesh.cell_size))
    U = scale * h * rng.standard_normal((dim + 1) * V)
    U[dim * V:] = np.clip(0.6 + 0.3 * rng.standard_normal(V), 0.05, 1)
    pt = np.clip(U[dim * V:] + 0.05 * rng.standard_normal(V), 0, 1)
    return LinearizationState(U=U, U_prev1=U, U_prev2=U, t=0.1, t_prev1=0.0, t_prev2=0.0, phi_tilde=pt), rng


@pytest.mark.parametrize("name,split,band", [("square", "none", 0.0), ("lshape", "miehe", 0.02),
                                             ("lshape3d", "none", 0.0), ("cube", "miehe", 0.02)])
def test_fd_jacobian_of_residual(name, split, band):
    """(A(U + s v) - A(U - s v)) / 2s == G~ v on unconstrained rows (phi_tilde fixed)."""
    from paper_1902_08112_b200 import model as M
    space = _space(name).finest
    st, rng = _state(space, 1, scale=0.1)
    n = st.U.size
    mask = M.ConstraintMask(np.zeros(n, bool), np.zeros(n))
    params = params_for(space, None, cls=M.MaterialParams)
    params.split_band = band
    sk = M.SplitKind.MIEHE if split == "miehe" else M.SplitKind.NOSPLIT
    v = rng.standard_normal(n)
    v[: n - space.mesh.n_vertices] *= float(np.min(space.mesh.cell_size)) * 0.1
    s = 1e-6
    rp = M.residual(space, st.with_U(st.U + s * v), mask, params, sk)
    rm = M.residual(space, st.with_U(st.U - s * v), mask, params, sk)
    fd = (rp - rm) / (2 * s)
    Gv = M.PhaseFieldOperator(space, st, mask, params, sk).apply(v)
    assert rel_err(Gv, fd) <= 1e-5


def test_vcycle_zero_linearity_and_constraints():
    from paper_1902_08112_b200 import mgsolve
    from paper_1902_08112_b200 import model as M
    disc = _space("cfg1")
    space = disc.finest
    st, rng = _state(space, 2)
    n = st.U.size
    flags = rng.random(n) < 0.1
    params = params_for(space, None, cls=M.MaterialParams)
    ctxs = mgsolve.build_level_contexts(disc, st, np.zeros(n, bool), M.ConstraintMask(flags, np.zeros(n)),
                                        params, M.SplitKind.NOSPLIT)
    FULL = mgsolve.PreconditionerKind.FULL
    z = mgsolve.vcycle(ctxs, FULL, np.zeros(n))
    assert np.all(z == 0.0)
    a, b = rng.standard_normal(n), rng.standard_normal(n)
    va, vb = mgsolve.vcycle(ctxs, FULL, a), mgsolve.vcycle(ctxs, FULL, b)
    vab = mgsolve.vcycle(ctxs, FULL, 2.0 * a - 3.0 * b)
    assert rel_err(vab, 2.0 * va - 3.0 * vb) <= 1e-12
    assert np.all(va[flags] == 0.0)
    a2 = a.copy()
    a2[flags] = 1e3 * rng.standard_normal(flags.sum())          # constrained input entries are ignored
    assert np.array_equal(mgsolve.vcycle(ctxs, FULL, a2), va)


def test_gmres_h_robust():
    """GMRES iteration counts stay within +-2 over refinements (tests/test_mgsolve.py:342-363)."""
    from paper_1902_08112_b200 import configs, krylov, mgsolve
    from paper_1902_08112_b200 import model as M
    its = []
    for levels in (4, 5, 6, 7):
        prob = configs.notched_square(levels, 4, "cfg1")
        ctxs = mgsolve.build_level_contexts(prob.disc, prob.state, prob.active, prob.dirichlet, prob.params,
                                            M.SplitKind.NOSPLIT)
        b = configs.fallback_rhs(prob)
        ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=200)
        _, k = krylov.gmres(ctxs[-1].op.apply, mgsolve.VCyclePreconditioner(ctxs), b, ctl)
        its.append(k)
    assert max(its) - min(its) <= 2, its


@pytest.mark.parametrize("name", ["square", "cube", "lshape"])
def test_all_constrained_is_identity(name):
    from paper_1902_08112_b200 import model as M
    space = _space(name).finest
    st, rng = _state(space, 3)
    n = st.U.size
    mask = M.ConstraintMask(np.ones(n, bool), np.zeros(n))
    params = params_for(space, None, cls=M.MaterialParams)
    op = M.PhaseFieldOperator(space, st, mask, params, M.SplitKind.NOSPLIT)
    v = rng.standard_normal(n)
    assert np.array_equal(op.apply(v), v)
    assert np.all(op.diagonal() == 1.0)
    assert np.all(M.residual(space, st, mask, params, M.SplitKind.NOSPLIT) == 0.0)


@pytest.mark.parametrize("dim", [2, 3])
def test_one_cell_mesh_and_one_level_hierarchy(dim):
    """The smallest inputs: a single cell, a hierarchy with one level (coarse solve only)."""
    from oracle import fe, jacobian, meshgen
    from paper_1902_08112_b200 import krylov, mgsolve
    from paper_1902_08112_b200 import model as M
    from paper_1902_08112_b200.fem import Discretization, build_hierarchy
    blocks = [[(0.0,) * dim, (1.0,) * dim]]
    disc = Discretization(build_hierarchy(blocks, 1, dim))
    space = disc.finest
    st, rng = _state(space, 4)
    n = st.U.size
    V = space.mesh.n_vertices
    flags = np.zeros(n, bool)
    face = [v for v in range(V) if v % 2 == 0]               # the x = 0 face: no rigid modes left
    for c in range(dim):
        flags[c * V + np.array(face)] = True
    mask = M.ConstraintMask(flags, np.zeros(n))
    params = params_for(space, None, cls=M.MaterialParams)
    op = M.PhaseFieldOperator(space, st, mask, params, M.SplitKind.NOSPLIT)
    T = fe.LevelTables(meshgen.build_hierarchy(blocks, 1, dim)[0], 0)
    ref = jacobian.JacobianOperator(T, jacobian.State(U=st.U, U_prev1=st.U, U_prev2=st.U, t=0.1, t_prev1=0.0,
                                                      t_prev2=0.0, phi_tilde=st.phi_tilde),
                                    flags, params_for(T, None, cls=jacobian.Material))
    v = rng.standard_normal(n)
    assert rel_err(op.apply(v), ref.apply(v)) <= 1e-12
    assert rel_err(op.diagonal(), ref.diagonal()) <= 1e-12
    ctxs = mgsolve.build_level_contexts(disc, st, np.zeros(n, bool), mask, params, M.SplitKind.NOSPLIT)
    assert len(ctxs) == 1
    r = rng.standard_normal(n)
    assert rel_err(mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, r),
                   mgsolve.coarse_solve(ctxs[0], np.where(flags, 0.0, r))) <= 1e-12
    b = np.where(flags, 0.0, r)
    x, its = krylov.gmres(op.apply, mgsolve.VCyclePreconditioner(ctxs), b,
                          krylov.SolverControl(abs_tol=0.0, rel_tol=1e-10))
    assert np.linalg.norm(op.apply(x) - b) <= 1e-9 * np.linalg.norm(b)

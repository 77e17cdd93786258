"""Known-answer pins of the Q2 oracle (oracle/q2.py).  The reference has no
Q2 elements, so parity for BASELINE configs[2] is pinned by properties
instead of golden vectors: exactness on quadratics, rigid-body kernel,
symmetry, assembled-vs-matrix-free diagonal.  CPU only."""
import numpy as np
import pytest

from oracle import jacobian, q2
from tests.golden.specs import params_for


def quad(p):
    x, y = p[..., 0], p[..., 1]
    return 1.0 + 2.0 * x + 3.0 * y + 4.0 * x * x + 5.0 * x * y + 6.0 * y * y


def quad_grad(p):
    x, y = p[..., 0], p[..., 1]
    return np.stack([2.0 + 8.0 * x + 5.0 * y, 3.0 + 5.0 * x + 12.0 * y], axis=-1)


def test_partition_of_unity_and_quadratic_exactness():
    lev = q2.q2_hierarchy(-1.0, 2.0, 3, 1)[0]
    T = q2.Q2Tables(lev)
    assert np.allclose(T.N.sum(axis=1), 1.0, atol=1e-15)
    assert np.allclose(T.gradN.sum(axis=1), 0.0, atol=1e-13)
    assert np.isclose(T.JxW.sum() * lev.n_cells, 9.0, rtol=1e-14)
    f = quad(lev.nodes)
    loc = f[lev.cells]
    assert np.allclose(T.at_qp(loc), quad(T.qp_coords), rtol=1e-13)
    assert np.allclose(T.grad_at_qp(loc), quad_grad(T.qp_coords), rtol=1e-12)


def test_transfers_exact_on_quadratics():
    levels = q2.q2_hierarchy(0.0, 1.0, 2, 3)
    tr = q2.Q2Transfers(levels)
    for l in range(2):
        c, f = levels[l], levels[l + 1]
        assert np.allclose(tr.P[l] @ quad(c.nodes), quad(f.nodes), rtol=1e-13)
        assert np.array_equal(f.nodes[tr.inj[l]], c.nodes)
        vc = np.random.default_rng(l).standard_normal(3 * c.n_vertices)
        assert np.array_equal(tr.restrict_nodal(tr.prolongate(vc, l), l), vc)
        wf = np.random.default_rng(l + 9).standard_normal(3 * f.n_vertices)
        assert np.isclose(tr.prolongate(vc, l) @ wf, vc @ tr.restrict(wf, l), rtol=1e-12)


def _op(lev, split="none", seed=0, flags=None):
    T = q2.Q2Tables(lev)
    rng = np.random.default_rng(seed)
    n = T.n_dofs
    U = 1e-2 * rng.standard_normal(n)
    U[T.phi_slice] = np.clip(0.6 + 0.4 * rng.standard_normal(T.n_vertices), 0, 1)
    st = jacobian.State(U=U, U_prev1=U, U_prev2=U, t=0.1, t_prev1=0.0, t_prev2=0.0,
                        phi_tilde=U[T.phi_slice].copy())
    mat = params_for(T, None, cls=jacobian.Material)
    flags = np.zeros(n, bool) if flags is None else flags
    return T, jacobian.JacobianOperator(T, st, flags, mat, split)


def test_rigid_body_modes_in_elastic_kernel():
    lev = q2.q2_hierarchy(0.0, 2.0, 3, 1)[0]
    T, op = _op(lev)
    X = lev.nodes
    V = lev.n_vertices
    for rbm in (np.concatenate([np.ones(V), np.zeros(V)]), np.concatenate([np.zeros(V), np.ones(V)]),
                np.concatenate([-X[:, 1], X[:, 0]])):
        assert np.abs(op.apply_block(0, rbm)).max() <= 1e-12 * np.abs(rbm).max() * 1e3


@pytest.mark.parametrize("split", ["none", "miehe"])
def test_blocks_symmetric_and_diagonal_assembled(split):
    lev = q2.q2_hierarchy(0.0, 1.0, 2, 1)[0]
    flags = np.random.default_rng(3).random(3 * lev.n_vertices) < 0.1
    T, op = _op(lev, split, flags=flags)
    n = T.n_dofs
    A = np.stack([op.apply(np.eye(n)[i]) for i in range(n)], axis=1)
    d = T.dim * T.n_vertices
    Au, Ap = A[:d, :d], A[d:, d:]
    assert np.allclose(Au, Au.T, rtol=1e-12, atol=1e-12 * np.abs(Au).max())
    assert np.allclose(Ap, Ap.T, rtol=1e-12, atol=1e-12 * np.abs(Ap).max())
    assert np.allclose(op.diagonal(), np.diag(A), rtol=1e-12, atol=0)
    assert np.allclose(A[:d, d:], np.where(flags[:d, None], 0.0, 0.0))   # G_uphi = 0

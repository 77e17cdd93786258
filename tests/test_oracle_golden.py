"""Pin the CPU oracle (oracle/) against golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle import fe, jacobian, solvers
from tests.conftest import rel_err
from tests.golden.specs import MESHES
from tests.helpers import OP_TAGS, oracle_levels, oracle_material, oracle_stack, oracle_state


@pytest.mark.parametrize("name", list(MESHES))
def test_mesh_numbering_matches_reference(golden, name):
    g = golden["meshes"]
    levels = oracle_levels(name)
    for l, lev in enumerate(levels):
        assert np.array_equal(lev.keys, g[f"{name}/{l}/keys"])
        assert np.array_equal(lev.cells, g[f"{name}/{l}/cells"])
        assert np.array_equal(lev.cell_size, g[f"{name}/{l}/cell_size"])


@pytest.mark.parametrize("name", list(MESHES))
def test_transfer_matrices_and_injection_exact(golden, name):
    g = golden["meshes"]
    _, _, tr = oracle_stack(name)
    for l in range(len(tr.levels) - 1):
        P = tr.P[l].tocsr()
        P.sort_indices()
        import scipy.sparse as sp
        R = sp.csr_matrix((g[f"{name}/{l}/P_data"], g[f"{name}/{l}/P_indices"],
                           g[f"{name}/{l}/P_indptr"]), shape=P.shape)
        R.sort_indices()
        assert np.array_equal(P.indptr, R.indptr)
        assert np.array_equal(P.indices, R.indices)
        assert np.array_equal(P.data, R.data)              # weights exactly 1, 1/2, 1/4, 1/8
        assert np.array_equal(tr.inj[l], g[f"{name}/{l}/inj"])


@pytest.mark.parametrize("name,variant", OP_TAGS)
@pytest.mark.parametrize("split", ["none", "miehe"])
def test_operator_oracle_vs_reference(golden, name, variant, split):
    g = golden["operator"]
    tag = f"{name}/{split}/{variant}"
    if not g.has(f"{tag}/apply"):
        pytest.skip("no such golden case")
    _, tables, _ = oracle_stack(name)
    T = tables[-1]
    mat = oracle_material(T, variant == "modulus")
    st = oracle_state(g[f"{tag}/U"], g[f"{tag}/phi_tilde"], g[f"{tag}/t"])
    op = jacobian.JacobianOperator(T, st, g[f"{tag}/flags"], mat, split)
    v = g[f"{tag}/v"]
    d = T.dim * T.n_vertices
    assert rel_err(op.apply(v), g[f"{tag}/apply"]) <= 1e-12
    assert rel_err(op.apply_block(0, v[:d]), g[f"{tag}/apply_u"]) <= 1e-12
    assert rel_err(op.apply_block(1, v[d:]), g[f"{tag}/apply_phi"]) <= 1e-12
    assert rel_err(op.diagonal(), g[f"{tag}/diagonal"]) <= 1e-12
    res = jacobian.residual(T, st, g[f"{tag}/flags"], mat, split)
    assert rel_err(res, g[f"{tag}/residual"]) <= 1e-12


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("variant", ["plain", "masked"])
def test_operator_band_oracle_vs_reference(golden, name, variant):
    """Miehe split with the C^1 blend (split_band > 0, model.py:65-86)."""
    g = golden["operator_band"]
    tag = f"{name}/miehe_band/{variant}"
    _, tables, _ = oracle_stack(name)
    T = tables[-1]
    mat = oracle_material(T)
    mat.split_band = float(g[f"{tag}/band"])
    st = oracle_state(g[f"{tag}/U"], g[f"{tag}/phi_tilde"], g[f"{tag}/t"])
    op = jacobian.JacobianOperator(T, st, g[f"{tag}/flags"], mat, "miehe")
    v = g[f"{tag}/v"]
    d = T.dim * T.n_vertices
    assert rel_err(op.apply(v), g[f"{tag}/apply"]) <= 1e-12
    assert rel_err(op.apply_block(0, v[:d]), g[f"{tag}/apply_u"]) <= 1e-12
    assert rel_err(op.apply_block(1, v[d:]), g[f"{tag}/apply_phi"]) <= 1e-12
    assert rel_err(op.diagonal(), g[f"{tag}/diagonal"]) <= 1e-12
    res = jacobian.residual(T, st, g[f"{tag}/flags"], mat, "miehe")
    assert rel_err(res, g[f"{tag}/residual"]) <= 1e-12
    # the blend region is populated (otherwise this case pins nothing new)
    sp_ = T
    loc = sp_.gather(g[f"{tag}/U"])
    gu = sp_.vec_grad_at_qp(loc[:, :T.dim])
    w = np.linalg.eigvalsh(0.5 * (gu + np.swapaxes(gu, -1, -2)))
    assert np.mean(np.abs(w) < mat.split_band) > 0.05


def test_operator_threads_bitwise(golden):
    g = golden["operator"]
    tag = "cfg1/none/masked"
    _, tables, _ = oracle_stack("cfg1")
    st = oracle_state(g[f"{tag}/U"], g[f"{tag}/phi_tilde"], g[f"{tag}/t"])
    mat = oracle_material(tables[-1])
    a = jacobian.JacobianOperator(tables[-1], st, g[f"{tag}/flags"], mat, threads=1).apply(g[f"{tag}/v"])
    b = jacobian.JacobianOperator(tables[-1], st, g[f"{tag}/flags"], mat, threads=4).apply(g[f"{tag}/v"])
    assert np.array_equal(a, b)


@pytest.mark.parametrize("name", list(MESHES))
def test_transfers_oracle_vs_reference(golden, name):
    g = golden["transfers"]
    _, _, tr = oracle_stack(name)
    for l in range(len(tr.levels) - 1):
        assert rel_err(tr.restrict(g[f"{name}/{l}/vf"], l), g[f"{name}/{l}/restrict"]) <= 1e-14
        assert rel_err(tr.prolongate(g[f"{name}/{l}/vc"], l), g[f"{name}/{l}/prolongate"]) <= 1e-14
        assert np.array_equal(tr.restrict_nodal(g[f"{name}/{l}/vf"], l),
                              g[f"{name}/{l}/restrict_nodal"])


def _mg_levels(g, name):
    levels, tables, tr = oracle_stack(name)
    st = jacobian.State(U=g[f"{name}/U"], U_prev1=g[f"{name}/U_prev1"], U_prev2=g[f"{name}/U_prev2"],
                        t=float(g[f"{name}/times"][0]), t_prev1=float(g[f"{name}/times"][1]),
                        t_prev2=float(g[f"{name}/times"][2]), phi_tilde=g[f"{name}/phi_tilde"])
    mat = oracle_material(tables[-1])
    return solvers.build_levels(tr, tables, st, g[f"{name}/active"], g[f"{name}/dirichlet"],
                                mat, "none")


@pytest.mark.parametrize("name", ["square", "lshape", "lshape3d", "cfg1"])
def test_multigrid_oracle_vs_reference(golden, name):
    g = golden["multigrid"]
    if not g.exists():
        pytest.skip("multigrid golden not generated")
    levs = _mg_levels(g, name)
    for l, lev in enumerate(levs):
        assert np.array_equal(lev.constrained, g[f"{name}/{l}/constrained"])
        assert rel_err(lev.diag, g[f"{name}/{l}/diag"]) <= 1e-12
        sp = np.array([[s.lambda_min_hat, s.lambda_max_hat, s.fallback] for s in lev.spectra])
        assert np.allclose(sp, g[f"{name}/{l}/spectra"], rtol=1e-9, atol=0)
    r = g[f"{name}/r"]
    assert rel_err(solvers.vcycle(levs, r, "full"), g[f"{name}/vcycle_full"]) <= 1e-9
    assert rel_err(solvers.vcycle(levs, r, "full", degree=3), g[f"{name}/vcycle_full_deg3"]) <= 1e-9
    assert rel_err(solvers.vcycle(levs, r, "blockdiag"), g[f"{name}/vcycle_block"]) <= 1e-9
    fine = levs[-1]
    blk = fine.op.blocks[0]
    prm = solvers.smoother_range(fine.spectra[0], 4)
    ap = lambda vb: fine.op.apply_block(0, vb)  # noqa: E731
    b = g[f"{name}/cheb_b"]
    assert rel_err(solvers.chebyshev(ap, fine.diag[blk], prm, np.zeros_like(b), b),
                   g[f"{name}/cheb_zero"]) <= 1e-12
    assert rel_err(solvers.chebyshev(ap, fine.diag[blk], prm, g[f"{name}/cheb_x0"], b),
                   g[f"{name}/cheb_nonzero"]) <= 1e-12
    assert rel_err(solvers.coarse_solve(levs[0], g[f"{name}/coarse_r"]), g[f"{name}/coarse"]) <= 1e-9
    ctl = solvers.Control(abs_tol=0.0, rel_tol=1e-8)
    x, its = solvers.gmres(fine.op.apply, lambda v: solvers.vcycle(levs, v, "full"),
                           g[f"{name}/gmres_rhs"], ctl)
    assert abs(its - int(g[f"{name}/gmres_iters"])) <= 1
    assert rel_err(x, g[f"{name}/gmres_x"]) <= 1e-6


def test_krylov_oracle_vs_reference(golden):
    g = golden["krylov"]
    K, b = g["K"], g["b"]
    x, its = solvers.gmres(lambda v: K @ v, None, b, solvers.Control(abs_tol=1e-13, rel_tol=1e-13))
    assert its == int(g["iters"])
    assert rel_err(x, g["x"]) <= 1e-12
    A = g["lap1d"]
    est = np.array([[e.lambda_min_hat, e.lambda_max_hat] for e in
                    (solvers.estimate_spectrum(lambda v: A @ v, np.diag(A), 10, s) for s in range(5))])
    assert np.allclose(est, g["lap1d_est"], rtol=1e-12)


@pytest.mark.parametrize("name", list(MESHES))
def test_qoi_oracle_vs_reference(golden, name):
    """crack_energy / bulk_energy / fracture_volume (model.py:472-504)."""
    g = golden["qoi"]
    _, tables, _ = oracle_stack(name)
    T = tables[-1]
    U = g[f"{name}/U"]
    st = oracle_state(U, U[T.phi_slice], g[f"{name}/t"])
    for variant in ("plain", "modulus"):
        mat = oracle_material(T, variant == "modulus")
        assert abs(jacobian.crack_energy(T, U, mat) - g[f"{name}/{variant}/crack_energy"]) <= \
            1e-12 * abs(g[f"{name}/{variant}/crack_energy"])
        assert abs(jacobian.fracture_volume(T, U) - g[f"{name}/{variant}/fracture_volume"]) <= \
            1e-12 * abs(g[f"{name}/{variant}/fracture_volume"])
        for split in ("none", "miehe"):
            ref = g[f"{name}/{variant}/{split}/bulk_energy"]
            assert abs(jacobian.bulk_energy(T, st, mat, split) - ref) <= 1e-12 * abs(ref)
        mat.split_band = 0.05
        ref = g[f"{name}/{variant}/miehe_band/bulk_energy"]
        assert abs(jacobian.bulk_energy(T, st, mat, "miehe") - ref) <= 1e-12 * abs(ref)

"""BASELINE configurations end to end on the GPU: vmult and one Newton-step
GMRES(30)+GMG solve vs the reference's golden outputs (cfg1; cfg2 at 256^2),
and size-independent properties at full cfg2 size (1024^2)."""
import numpy as np
import pytest
import torch

from tests.conftest import rel_err

pytestmark = pytest.mark.gpu


def _setup(name, levels=None):
    from paper_1902_08112_b200 import configs
    from paper_1902_08112_b200.model import ConstraintMask, PhaseFieldOperator, SplitKind
    prob = configs.make(name, levels)
    mask = prob.dirichlet.combined_with(prob.active, np.zeros(prob.n_dofs))
    op = PhaseFieldOperator(prob.disc.finest, prob.state, ConstraintMask(mask.is_constrained,
                                                                         mask.inhomogeneity),
                            prob.params, SplitKind.NOSPLIT)
    return prob, mask, op


@pytest.mark.parametrize("name,levels,tag", [("cfg1", None, "cfg1"), ("cfg2", 6, "cfg2_l6")])
def test_config_vmult_and_solve_match_reference(golden, name, levels, tag):
    from paper_1902_08112_b200 import krylov, mgsolve
    from paper_1902_08112_b200.model import SplitKind
    g = golden["configs"]
    prob, mask, op = _setup(name, levels)
    chk = g[f"{tag}/checksum"]
    assert np.isclose(prob.state.U.sum(), chk[0], rtol=1e-13, atol=0)
    assert np.isclose(prob.v.sum(), chk[1], rtol=1e-13, atol=0)
    assert mask.is_constrained.sum() == chk[2]
    assert rel_err(op.apply(prob.v), g[f"{tag}/apply"]) <= 1e-12
    assert rel_err(op.diagonal(), g[f"{tag}/diagonal"]) <= 1e-12
    ctxs = mgsolve.build_level_contexts(prob.disc, prob.state, prob.active, prob.dirichlet,
                                        prob.params, SplitKind.NOSPLIT)
    for l, c in enumerate(ctxs):
        sp = np.array([[s.lambda_min_hat, s.lambda_max_hat, s.fallback] for s in c.spectra])
        assert np.allclose(sp, g[f"{tag}/{l}/spectra"], rtol=1e-10, atol=0)
    ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)
    pc = mgsolve.VCyclePreconditioner(ctxs, mgsolve.PreconditionerKind.FULL, degree=prob.degree)
    x, its = krylov.gmres(ctxs[-1].op.apply, pc, g[f"{tag}/gmres_rhs"], ctl)
    assert abs(its - int(g[f"{tag}/gmres_iters"])) <= 1, (its, int(g[f"{tag}/gmres_iters"]))
    assert rel_err(x, g[f"{tag}/gmres_x"]) <= 1e-6


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4", "cfg5"])
def test_full_size_properties(name):
    """BASELINE sizes (cfg5: 228M DoFs, the largest): linearity, identity rows,
    symmetry of the u block, determinism, and the residual's constrained rows."""
    from paper_1902_08112_b200 import model as M
    prob, mask, op = _setup(name)
    n, d = op.n_dofs, op.dim * op.V
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(n, device="cuda", dtype=torch.float64, generator=g)
    y = torch.randn(n, device="cuda", dtype=torch.float64, generator=g)
    ax, ay = op.apply(x), op.apply(y)
    assert torch.equal(ax, op.apply(x))
    lin = op.apply(x + 0.5 * y)
    assert (lin - (ax + 0.5 * ay)).norm() <= 1e-13 * lin.norm()
    c = torch.as_tensor(mask.is_constrained, device="cuda")
    assert torch.equal(ax[c], x[c])
    xu, yu = x[:d].clone(), y[:d].clone()
    xu[c[:d]] = 0
    yu[c[:d]] = 0
    lhs = torch.dot(op.apply_block(0, xu), yu)
    rhs = torch.dot(xu, op.apply_block(0, yu))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    R = M.residual(prob.disc.finest, M.LinearizationState(
        U=torch.as_tensor(prob.state.U, device="cuda"), U_prev1=None, U_prev2=None, t=prob.state.t,
        t_prev1=prob.state.t_prev1, t_prev2=prob.state.t_prev2,
        phi_tilde=torch.as_tensor(prob.state.phi_tilde, device="cuda")), prob.dirichlet, prob.params,
        M.SplitKind.NOSPLIT)
    assert torch.isfinite(R).all()
    dc = torch.as_tensor(prob.dirichlet.is_constrained, device="cuda")
    assert torch.all(R[dc] == 0.0)


@pytest.mark.parametrize("name,levels,tag", [("cfg1", None, "cfg1"), ("cfg2", 6, "cfg2_l6")])
def test_newton_rhs_on_gpu_matches_reference(golden, name, levels, tag):
    """R~ = -A(U) with constrained rows zeroed (nonlinear.py:146-160) from the GPU residual."""
    from paper_1902_08112_b200 import model as M
    g = golden["configs"]
    prob, mask, op = _setup(name, levels)
    R = -M.residual(prob.disc.finest, prob.state, prob.dirichlet, prob.params, M.SplitKind.NOSPLIT)
    R[mask.is_constrained] = 0.0
    assert rel_err(R, g[f"{tag}/gmres_rhs"]) <= 1e-12


def test_cfg3_q2_newton_step_matches_oracle():
    """cfg3 (Q2, pressure) at 4 levels (64^2 Q2 cells): Newton RHS, level
    contexts, and the GMRES iteration count against the Q2 oracle."""
    from oracle import jacobian, q2, solvers
    from paper_1902_08112_b200 import krylov, mgsolve
    from paper_1902_08112_b200 import model as M
    prob, mask, op = _setup("cfg3", 4)
    levels = q2.q2_hierarchy(-20.0, 20.0, 8, 4)
    tables = [q2.Q2Tables(lev, l) for l, lev in enumerate(levels)]
    tr = q2.Q2Transfers(levels)
    p = prob.params
    mat = jacobian.Material(mu=p.mu, lam=p.lam, g_c=p.g_c, kappa=p.kappa, eps=p.eps,
                            pressure_fn=p.pressure_fn)
    s = prob.state
    st = jacobian.State(U=s.U, U_prev1=s.U_prev1, U_prev2=s.U_prev2, t=s.t, t_prev1=s.t_prev1,
                        t_prev2=s.t_prev2, phi_tilde=s.phi_tilde)
    R_ref = -jacobian.residual(tables[-1], st, prob.dirichlet.is_constrained, mat)
    R_ref[mask.is_constrained] = 0.0
    R = -M.residual(prob.disc.finest, s, prob.dirichlet, p, M.SplitKind.NOSPLIT)
    R[mask.is_constrained] = 0.0
    assert rel_err(R, R_ref) <= 1e-12
    olev = solvers.build_levels(tr, tables, st, prob.active, prob.dirichlet.is_constrained, mat, "none")
    ctxs = mgsolve.build_level_contexts(prob.disc, s, prob.active, prob.dirichlet, p, M.SplitKind.NOSPLIT)
    for c, o in zip(ctxs, olev):
        assert np.array_equal(c.constrained, o.constrained)
        assert rel_err(c.diag, o.diag) <= 1e-12
    ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)
    x, its = krylov.gmres(ctxs[-1].op.apply, mgsolve.VCyclePreconditioner(ctxs, degree=prob.degree), R, ctl)
    xo, its_o = solvers.gmres(olev[-1].op.apply, lambda v: solvers.vcycle(olev, v, "full", degree=prob.degree),
                              R_ref, solvers.Control(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000))
    assert abs(its - its_o) <= 1, (its, its_o)
    assert rel_err(x, xo) <= 1e-6

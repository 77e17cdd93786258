"""GPU transfers, level contexts, Chebyshev smoother, V-cycle and GMRES vs the
reference's golden outputs.  Index maps and masks must be bit-exact; vectors
within the stated relative tolerances; GMRES iteration counts equal +-1."""
import numpy as np
import pytest
import torch

from tests.conftest import rel_err
from tests.golden.specs import MESHES
from tests.helpers import product_disc, product_params, product_state

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", list(MESHES))
def test_transfers_match_reference(golden, name):
    g, gm = golden["transfers"], golden["meshes"]
    disc = product_disc(name)
    for l in range(disc.hierarchy.n_levels - 1):
        assert np.array_equal(disc.injection(l), gm[f"{name}/{l}/inj"])
        assert rel_err(disc.restrict(g[f"{name}/{l}/vf"], l), g[f"{name}/{l}/restrict"]) <= 1e-14
        assert rel_err(disc.prolongate(g[f"{name}/{l}/vc"], l), g[f"{name}/{l}/prolongate"]) <= 1e-14
        assert np.array_equal(disc.restrict_nodal(g[f"{name}/{l}/vf"], l),
                              g[f"{name}/{l}/restrict_nodal"])


def test_transfer_size_checks_raise():
    disc = product_disc("square")
    with pytest.raises(ValueError):
        disc.prolongate(np.zeros(5), 0)
    with pytest.raises(ValueError):
        disc.restrict(np.zeros(5), 0)


@pytest.mark.parametrize("name", ["cube", "lprism", "lshape"])
def test_transfer_adjointness(name):
    disc = product_disc(name)
    rng = np.random.default_rng(1)
    for l in range(disc.hierarchy.n_levels - 1):
        Vc = disc.hierarchy.levels[l].n_vertices
        Vf = disc.hierarchy.levels[l + 1].n_vertices
        vc, wf = rng.standard_normal(Vc), rng.standard_normal(Vf)
        lhs = disc.prolongate_scalar(vc, l) @ wf
        rhs = vc @ disc.restrict_scalar(wf, l)
        assert abs(lhs - rhs) <= 1e-13 * abs(lhs)


def _contexts(g, name, miehe=False):
    from paper_1902_08112_b200 import mgsolve
    from paper_1902_08112_b200.model import ConstraintMask, SplitKind
    disc = product_disc(name)
    t = g[f"{name}/times"]
    st = product_state(g[f"{name}/U"], g[f"{name}/phi_tilde"], t[0], g[f"{name}/U_prev1"],
                       g[f"{name}/U_prev2"], t[1], t[2])
    dirichlet = ConstraintMask(g[f"{name}/dirichlet"], g[f"{name}/dirichlet_vals"])
    params = product_params(disc.finest)
    if miehe:
        params.split_band = float(g[f"{name}/band"])
    ctxs = mgsolve.build_level_contexts(disc, st, g[f"{name}/active"], dirichlet, params,
                                        SplitKind.MIEHE if miehe else SplitKind.NOSPLIT)
    return disc, ctxs


@pytest.mark.parametrize("name", ["lshape", "lshape3d"])
def test_miehe_contexts_vcycle_gmres(golden, name):
    """Miehe split through the whole solve: level diagonals and spectra, the
    V-cycle and the GMRES iteration count vs the reference."""
    from paper_1902_08112_b200 import krylov, mgsolve
    g = golden["multigrid_miehe"]
    disc, ctxs = _contexts(g, name, miehe=True)
    for l, c in enumerate(ctxs):
        assert np.array_equal(c.constrained, g[f"{name}/{l}/constrained"])
        assert rel_err(c.diag, g[f"{name}/{l}/diag"]) <= 1e-12
        sp = np.array([[s.lambda_min_hat, s.lambda_max_hat, s.fallback] for s in c.spectra])
        assert np.allclose(sp, g[f"{name}/{l}/spectra"], rtol=1e-10, atol=0), (l, sp)
    FULL = mgsolve.PreconditionerKind.FULL
    assert rel_err(mgsolve.vcycle(ctxs, FULL, g[f"{name}/r"]), g[f"{name}/vcycle_full"]) <= 1e-10
    ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)
    x, its = krylov.gmres(ctxs[-1].op.apply, mgsolve.VCyclePreconditioner(ctxs, FULL),
                          g[f"{name}/gmres_rhs"], ctl)
    assert abs(its - int(g[f"{name}/gmres_iters"])) <= 1
    assert rel_err(x, g[f"{name}/gmres_x"]) <= 1e-6


MG = ["square", "lshape", "lshape3d", "cfg1"]


@pytest.mark.parametrize("name", MG)
def test_level_contexts(golden, name):
    g = golden["multigrid"]
    disc, ctxs = _contexts(g, name)
    for l, c in enumerate(ctxs):
        assert np.array_equal(c.constrained, g[f"{name}/{l}/constrained"])     # bit-exact masks
        assert rel_err(c.diag, g[f"{name}/{l}/diag"]) <= 1e-12
        sp = np.array([[s.lambda_min_hat, s.lambda_max_hat, s.fallback] for s in c.spectra])
        assert np.allclose(sp, g[f"{name}/{l}/spectra"], rtol=1e-10, atol=0), (l, sp)


@pytest.mark.parametrize("name", MG)
def test_vcycle_chebyshev_coarse(golden, name):
    from paper_1902_08112_b200 import mgsolve
    g = golden["multigrid"]
    disc, ctxs = _contexts(g, name)
    r = g[f"{name}/r"]
    FULL, BLK = mgsolve.PreconditionerKind.FULL, mgsolve.PreconditionerKind.BLOCK_DIAG
    out = mgsolve.vcycle(ctxs, FULL, r)
    assert rel_err(out, g[f"{name}/vcycle_full"]) <= 1e-10
    assert np.all(out[ctxs[-1].constrained] == 0.0)
    assert rel_err(mgsolve.vcycle(ctxs, FULL, r, degree=3), g[f"{name}/vcycle_full_deg3"]) <= 1e-10
    assert rel_err(mgsolve.vcycle(ctxs, BLK, r), g[f"{name}/vcycle_block"]) <= 1e-10
    fine = ctxs[-1]
    blk = fine.op.blocks[0]
    prm = mgsolve.smoother_params(fine.spectra[0], 4)
    b = g[f"{name}/cheb_b"]
    ap = lambda vb: fine.op.apply_block(0, vb)  # noqa: E731
    assert rel_err(mgsolve.chebyshev_apply(ap, fine.diag[blk], prm, np.zeros_like(b), b),
                   g[f"{name}/cheb_zero"]) <= 1e-10
    assert rel_err(mgsolve.chebyshev_apply(ap, fine.diag[blk], prm, g[f"{name}/cheb_x0"], b),
                   g[f"{name}/cheb_nonzero"]) <= 1e-10
    assert rel_err(mgsolve.coarse_solve(ctxs[0], g[f"{name}/coarse_r"]), g[f"{name}/coarse"]) <= 1e-10


@pytest.mark.parametrize("name", MG)
def test_vcycle_graph_equals_eager(golden, name, monkeypatch):
    from paper_1902_08112_b200 import mgsolve
    g = golden["multigrid"]
    disc, ctxs = _contexts(g, name)
    r = torch.as_tensor(g[f"{name}/r"], device="cuda")
    a = mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, r)
    b = mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, r)   # graph replay
    cyc = mgsolve._NativeCycle.get(ctxs, 4, 1e-3, 30)
    cyc.use_graph = False
    c = mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, r)
    assert torch.equal(a, b) and torch.equal(a, c)


@pytest.mark.parametrize("name", MG)
def test_gmres_newton_step(golden, name):
    from paper_1902_08112_b200 import krylov, mgsolve
    g = golden["multigrid"]
    disc, ctxs = _contexts(g, name)
    ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)
    pc = mgsolve.VCyclePreconditioner(ctxs, mgsolve.PreconditionerKind.FULL)
    x, its = krylov.gmres(ctxs[-1].op.apply, pc, g[f"{name}/gmres_rhs"], ctl)
    assert abs(its - int(g[f"{name}/gmres_iters"])) <= 1
    assert rel_err(x, g[f"{name}/gmres_x"]) <= 1e-6
    # the reference's lambda form of the preconditioner gives the same answer
    x2, its2 = krylov.gmres(ctxs[-1].op.apply,
                            lambda v: mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, v),
                            g[f"{name}/gmres_rhs"], ctl)
    assert its2 == its and rel_err(x2, x) <= 1e-13


def test_generic_krylov_on_numpy_operators(golden):
    from paper_1902_08112_b200 import krylov
    g = golden["krylov"]
    K, b = g["K"], g["b"]
    x, its = krylov.gmres(lambda v: K @ v, None, b,
                          krylov.SolverControl(abs_tol=1e-13, rel_tol=1e-13))
    assert isinstance(x, np.ndarray)
    assert abs(its - int(g["iters"])) <= 1
    assert rel_err(x, g["x"]) <= 1e-10
    A = g["lap1d"]
    est = np.array([[e.lambda_min_hat, e.lambda_max_hat] for e in
                    (krylov.estimate_spectrum(lambda v: A @ v, np.diag(A), 10, s) for s in range(5))])
    assert np.allclose(est, g["lap1d_est"], rtol=1e-10)
    e = krylov.estimate_spectrum(lambda v: v, np.ones(12), seed=3)
    assert e.fallback and e.lambda_min_hat == e.lambda_max_hat == 1.0
    x, its = krylov.gmres(lambda v: 2 * v, None, np.zeros(5))
    assert its == 0 and not x.any()
    with pytest.raises(krylov.NoConvergence) as ei:
        krylov.gmres(lambda v: K @ v, None, np.ones(9),
                     krylov.SolverControl(abs_tol=0, rel_tol=1e-14, max_iters=2, restart=2))
    assert ei.value.iterations == 2


def test_generic_vcycle_on_model_problem(golden):
    """contexts_from_operators + vcycle over a non-native (numpy) operator."""
    from paper_1902_08112_b200 import mgsolve
    from tests.modelproblem import build_model_problem
    disc = product_disc("square")
    ops = build_model_problem(disc, eps=1.0)
    ctxs = mgsolve.contexts_from_operators(disc, ops)
    rng = np.random.default_rng(0)
    n = disc.finest.dofmap.n_dofs
    r1, r2 = rng.standard_normal(n), rng.standard_normal(n)
    lhs = mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, r1 + 0.5 * r2)
    rhs = (mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, r1)
           + 0.5 * mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, r2))
    assert rel_err(lhs, rhs) <= 1e-12
    assert np.all(lhs[ctxs[-1].constrained] == 0.0)


def test_setup_reuse_across_newton_steps(golden, monkeypatch):
    """Reusable setup (mgsolve._Session): a second build on the same hierarchy
    with a different state replays the recorded graphs and gives bit-identical
    results to a from-scratch build; contexts of the first build stay valid
    (detached onto private buffers) and keep giving their own results."""
    from paper_1902_08112_b200 import krylov, mgsolve
    from paper_1902_08112_b200.model import ConstraintMask, SplitKind
    g = golden["multigrid"]
    name = "cfg1"
    disc = product_disc(name)
    t = g[f"{name}/times"]
    dirichlet = ConstraintMask(g[f"{name}/dirichlet"], g[f"{name}/dirichlet_vals"])
    params = product_params(disc.finest)
    rng = np.random.default_rng(4)
    U2 = g[f"{name}/U"] + 1e-3 * rng.standard_normal(g[f"{name}/U"].size)
    states = [product_state(U, g[f"{name}/phi_tilde"], t[0], g[f"{name}/U_prev1"],
                            g[f"{name}/U_prev2"], t[1], t[2]) for U in (g[f"{name}/U"], U2)]
    r = torch.as_tensor(g[f"{name}/r"], device="cuda")
    FULL = mgsolve.PreconditionerKind.FULL

    def build(st):
        return mgsolve.build_level_contexts(disc, st, g[f"{name}/active"], dirichlet, params,
                                            SplitKind.NOSPLIT)

    monkeypatch.setattr(mgsolve, "REUSE_SETUP", False)
    fresh = []
    for st in states:
        c = build(st)
        fresh.append((mgsolve.vcycle(c, FULL, r), [cc.spectra for cc in c], c[-1].op.apply(r)))
    monkeypatch.setattr(mgsolve, "REUSE_SETUP", True)
    mgsolve._Session._cache.clear()
    c1 = build(states[0])
    v1 = mgsolve.vcycle(c1, FULL, r)
    c2 = build(states[1])                     # same session: replay, c1 detached
    assert c2[-1]._session is not None and c1[-1]._session is None
    v2 = mgsolve.vcycle(c2, FULL, r)
    assert torch.equal(v1, fresh[0][0]) and torch.equal(v2, fresh[1][0])
    assert [cc.spectra for cc in c2] == fresh[1][1]
    assert torch.equal(c2[-1].op.apply(r), fresh[1][2])
    # detached first-build contexts still see the first state
    assert torch.equal(mgsolve.vcycle(c1, FULL, r), fresh[0][0])
    assert torch.equal(c1[-1].op.apply(r), fresh[0][2])
    # a third build (back to state 0) replays again and matches
    c3 = build(states[0])
    assert torch.equal(mgsolve.vcycle(c3, FULL, r), fresh[0][0])
    ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)
    x, its = krylov.gmres(c3[-1].op.apply, mgsolve.VCyclePreconditioner(c3, FULL),
                          g[f"{name}/gmres_rhs"], ctl)
    assert abs(its - int(g[f"{name}/gmres_iters"])) <= 1


@pytest.mark.parametrize("name", MG)
def test_blockdiag_smoothing_matches_per_block(golden, name, monkeypatch):
    """One block-diagonal kernel per Chebyshev step == the per-block kernels."""
    from paper_1902_08112_b200 import mgsolve
    g = golden["multigrid"]
    r = torch.as_tensor(g[f"{name}/r"], device="cuda")
    FULL = mgsolve.PreconditionerKind.FULL
    out = []
    for flag in (True, False):
        monkeypatch.setattr(mgsolve, "BLOCKDIAG_SMOOTH", flag)
        mgsolve._Session._cache.clear()
        disc, ctxs = _contexts(g, name)
        out.append(mgsolve.vcycle(ctxs, FULL, r).cpu().numpy())
    assert rel_err(out[0], out[1]) <= 1e-12


@pytest.mark.parametrize("name", MG)
def test_coarse_kernel_matches_per_step(golden, name, monkeypatch):
    """Single-launch coarse solve (pffmg_coarse_cheb) == the per-step kernels."""
    from paper_1902_08112_b200 import mgsolve
    g = golden["multigrid"]
    rc = g[f"{name}/coarse_r"]
    r = torch.as_tensor(g[f"{name}/r"], device="cuda")
    out = []
    for flag in (True, False):
        monkeypatch.setattr(mgsolve, "COARSE_KERNEL", flag)
        mgsolve._Session._cache.clear()
        disc, ctxs = _contexts(g, name)
        out.append((mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, r).cpu().numpy(),
                    mgsolve.coarse_solve(ctxs[0], rc)))
    assert rel_err(out[0][0], out[1][0]) <= 1e-12
    assert rel_err(out[0][1], out[1][1]) <= 1e-12
    assert rel_err(out[0][1], g[f"{name}/coarse"]) <= 1e-10


@pytest.mark.parametrize("name", MG)
def test_fused_descent_and_entry_match_separate_kernels(golden, name, monkeypatch):
    """pffmg_restrict_init_bd (fused descent) and pffmg_masked_copy_init_bd (fused
    V-cycle entry) are bitwise the separate kernels they replace."""
    from paper_1902_08112_b200 import mgsolve
    g = golden["multigrid"]
    r = torch.as_tensor(g[f"{name}/r"], device="cuda")
    out = []
    for flag in (True, False):
        monkeypatch.setattr(mgsolve, "FUSED_DESCENT", flag)
        mgsolve._Session._cache.clear()
        mgsolve._NativeCycle._cache.clear()
        disc, ctxs = _contexts(g, name)
        out.append(mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, r))
    assert torch.equal(out[0], out[1])


@pytest.mark.parametrize("name", MG)
@pytest.mark.parametrize("kind", ["full", "block_diag"])
@pytest.mark.parametrize("bd", [True, False])
def test_lean_chebyshev_start_matches_full_start(golden, name, kind, bd, monkeypatch):
    """x = 0 starts that store d only + pffmg_cheb_first_* (the first step reads r
    from the right-hand side and x from d) are bitwise the full start + step, in
    the block-diagonal and the per-block smoothers, FULL and BLOCK_DIAG cycles."""
    from paper_1902_08112_b200 import _lib, mgsolve
    g = golden["multigrid"]
    r = torch.as_tensor(g[f"{name}/r"], device="cuda")
    pk = mgsolve.PreconditionerKind.FULL if kind == "full" else mgsolve.PreconditionerKind.BLOCK_DIAG
    monkeypatch.setattr(mgsolve, "BLOCKDIAG_SMOOTH", bd)
    out, seen = [], []
    real = _lib.call
    monkeypatch.setattr(_lib, "call", lambda n_, *a: (seen.append(n_), real(n_, *a))[1])
    for flag in (True, False):
        monkeypatch.setattr(mgsolve, "LEAN_START", flag)
        mgsolve._Session._cache.clear()
        mgsolve._NativeCycle._cache.clear()
        seen.clear()
        disc, ctxs = _contexts(g, name)
        out.append(mgsolve.vcycle(ctxs, pk, r))
        assert any(n_.startswith("pffmg_cheb_first") for n_ in seen) == flag
    assert torch.equal(out[0], out[1])


def test_gmres_restart_above_64():
    """Restart lengths above the one-launch MGS bound (64) take the multi-launch
    Arnoldi path and still match the oracle (reference krylov.py:50-136 accepts any m)."""
    from oracle import solvers
    from paper_1902_08112_b200 import krylov
    rng = np.random.default_rng(5)
    n = 300
    A = np.diag(np.linspace(1.0, 400.0, n)) + 1e-3 * rng.standard_normal((n, n))
    b = rng.standard_normal(n)
    At = torch.as_tensor(A, device="cuda")
    ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-10, restart=100, max_iters=1000)
    x, its = krylov.gmres(lambda v: At @ v, None, b, ctl)
    xo, its_o = solvers.gmres(lambda v: A @ v, None, b,
                              solvers.Control(abs_tol=0.0, rel_tol=1e-10, restart=100, max_iters=1000))
    assert its > 64
    assert abs(its - its_o) <= 1
    assert rel_err(x, xo) <= 1e-8

"""Generate the golden fixtures of tests/golden/ from the REFERENCE itself.

Run in the build container only (it imports /root/reference/pkg/src):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every output below is computed by the unmodified reference `fracmg`
(meshes, transfers, PhaseFieldOperator.apply/apply_block/diagonal,
build_level_contexts, vcycle, chebyshev_apply, coarse_solve, gmres,
estimate_spectrum).  Inputs are stored alongside (or regenerated from seeds
and checked by checksum), so the GPU tests on a box without the reference
compare against these files.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from fracmg import fem, krylov, mesh, mgsolve, model, selfcheck  # noqa: E402
from fracmg.fem import ConstraintMask, Discretization  # noqa: E402
from fracmg.model import LinearizationState, MaterialParams, SplitKind  # noqa: E402

from tests.golden.specs import MESHES, face_tagger, modulus, params_for  # noqa: E402


def ref_hierarchy(spec):
    blocks, n_levels, dim = spec
    return mesh._build_hierarchy(blocks, n_levels, dim, lambda lo, hi, ax, sd: np.zeros(len(lo)))


def save(name, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"  wrote {name}.npz ({os.path.getsize(path) / 1024:.0f} KiB)")


def gen_meshes():
    out = {}
    for name, spec in MESHES.items():
        hier = ref_hierarchy(spec)
        disc = Discretization(hier)
        for l, lev in enumerate(hier.levels):
            out[f"{name}/{l}/keys"] = lev.keys.astype(np.int32)
            out[f"{name}/{l}/cells"] = lev.cells.astype(np.int32)
            out[f"{name}/{l}/cell_size"] = lev.cell_size
        for l in range(hier.n_levels - 1):
            P = disc._P[l].tocsr()
            out[f"{name}/{l}/P_data"] = P.data
            out[f"{name}/{l}/P_indices"] = P.indices.astype(np.int32)
            out[f"{name}/{l}/P_indptr"] = P.indptr.astype(np.int32)
            out[f"{name}/{l}/inj"] = disc.injection(l).astype(np.int64)
    save("meshes", **out)


def gen_operator():
    out = {}
    rng = np.random.default_rng(20261019)
    for name, spec in MESHES.items():
        disc = Discretization(ref_hierarchy(spec))
        space = disc.finest
        n = space.dofmap.n_dofs
        for split in (SplitKind.NOSPLIT, SplitKind.MIEHE):
            for variant in ("plain", "masked", "modulus"):
                if split is SplitKind.MIEHE and variant == "modulus":
                    continue
                tag = f"{name}/{split.value}/{variant}"
                params = params_for(space, modulus if variant == "modulus" else None)
                try:
                    state = selfcheck.random_state(space, rng, t=0.1,
                                                   gapped=split is SplitKind.MIEHE)
                except RuntimeError:      # large meshes: a fully gapped sample is unlikely
                    state = selfcheck.random_state(space, rng, t=0.1)
                flags = (rng.random(n) < 0.15) if variant == "masked" else np.zeros(n, bool)
                mask = ConstraintMask(flags, np.zeros(n))
                v = rng.standard_normal(n)
                op = model.PhaseFieldOperator(space, state, mask, params, split)
                d = space.dim * space.dofmap.n_vertices
                out[f"{tag}/U"] = state.U
                out[f"{tag}/phi_tilde"] = state.phi_tilde
                out[f"{tag}/t"] = np.array(state.t)
                out[f"{tag}/flags"] = flags
                out[f"{tag}/v"] = v
                out[f"{tag}/apply"] = op.apply(v)
                out[f"{tag}/apply_u"] = op.apply_block(0, v[:d])
                out[f"{tag}/apply_phi"] = op.apply_block(1, v[d:])
                out[f"{tag}/diagonal"] = op.diagonal()
                out[f"{tag}/residual"] = model.residual(space, state, mask, params, split)
    save("operator", **out)


def gen_operator_band():
    """Miehe split with the C^1 blend (MaterialParams.split_band > 0): band
    0.05 is about half the typical principal strain of random_state, so many
    quadrature points sit inside the blend (model.py:65-86)."""
    out = {}
    rng = np.random.default_rng(20261020)
    for name, spec in MESHES.items():
        disc = Discretization(ref_hierarchy(spec))
        space = disc.finest
        n = space.dofmap.n_dofs
        for variant in ("plain", "masked"):
            tag = f"{name}/miehe_band/{variant}"
            params = params_for(space, None)
            params.split_band = 0.05
            state = selfcheck.random_state(space, rng, t=0.1)
            flags = (rng.random(n) < 0.15) if variant == "masked" else np.zeros(n, bool)
            mask = ConstraintMask(flags, np.zeros(n))
            v = rng.standard_normal(n)
            split = SplitKind.MIEHE
            op = model.PhaseFieldOperator(space, state, mask, params, split)
            d = space.dim * space.dofmap.n_vertices
            out[f"{tag}/band"] = np.array(params.split_band)
            out[f"{tag}/U"] = state.U
            out[f"{tag}/phi_tilde"] = state.phi_tilde
            out[f"{tag}/t"] = np.array(state.t)
            out[f"{tag}/flags"] = flags
            out[f"{tag}/v"] = v
            out[f"{tag}/apply"] = op.apply(v)
            out[f"{tag}/apply_u"] = op.apply_block(0, v[:d])
            out[f"{tag}/apply_phi"] = op.apply_block(1, v[d:])
            out[f"{tag}/diagonal"] = op.diagonal()
            out[f"{tag}/residual"] = model.residual(space, state, mask, params, split)
    save("operator_band", **out)


def gen_qoi():
    """crack_energy / bulk_energy / fracture_volume (model.py:472-504) on every
    mesh, both splits (blended Miehe too), with and without a modulus field."""
    out = {}
    rng = np.random.default_rng(20261021)
    for name, spec in MESHES.items():
        disc = Discretization(ref_hierarchy(spec))
        space = disc.finest
        state = selfcheck.random_state(space, rng, t=0.1)
        out[f"{name}/U"] = state.U
        out[f"{name}/t"] = np.array(state.t)
        for variant in ("plain", "modulus"):
            params = params_for(space, modulus if variant == "modulus" else None)
            out[f"{name}/{variant}/crack_energy"] = np.array(model.crack_energy(space, state, params))
            out[f"{name}/{variant}/fracture_volume"] = np.array(model.fracture_volume(space, state.U))
            for split in (SplitKind.NOSPLIT, SplitKind.MIEHE):
                out[f"{name}/{variant}/{split.value}/bulk_energy"] = np.array(
                    model.bulk_energy(space, state, params, split))
            params.split_band = 0.05
            out[f"{name}/{variant}/miehe_band/bulk_energy"] = np.array(
                model.bulk_energy(space, state, params, SplitKind.MIEHE))
    save("qoi", **out)


def gen_boundary():
    """boundary_load (model.py:511-547) on every mesh with the face_tagger tags:
    every tag x direction, NoSplit / Miehe / blended Miehe, with and without a
    modulus field; plus the reference's boundary-face arrays."""
    out = {}
    rng = np.random.default_rng(20261022)
    for name, (blocks, n_levels, dim) in MESHES.items():
        hier = mesh._build_hierarchy(blocks, n_levels, dim, face_tagger)
        disc = Discretization(hier)
        space = disc.finest
        m = space.mesh
        out[f"{name}/bf_cell"] = m.bf_cell
        out[f"{name}/bf_face"] = m.bf_face
        out[f"{name}/bf_tag"] = m.bf_tag
        state = selfcheck.random_state(space, rng, t=0.1)
        out[f"{name}/U"] = state.U
        for variant in ("plain", "modulus"):
            params = params_for(space, modulus if variant == "modulus" else None)
            for split, band in ((SplitKind.NOSPLIT, 0.0), (SplitKind.MIEHE, 0.0), (SplitKind.MIEHE, 0.05)):
                params.split_band = band
                key = split.value + ("_band" if band else "")
                vals = np.array([[model.boundary_load(space, state, params, split, tag, d)
                                  for d in range(dim)] for tag in range(4)])
                out[f"{name}/{variant}/{key}/load"] = vals
    save("boundary", **out)


def gen_transfers():
    out = {}
    rng = np.random.default_rng(99)
    for name, spec in MESHES.items():
        hier = ref_hierarchy(spec)
        disc = Discretization(hier)
        nc = hier.dim + 1
        for l in range(hier.n_levels - 1):
            Vc, Vf = hier.levels[l].n_vertices, hier.levels[l + 1].n_vertices
            vf = rng.standard_normal(nc * Vf)
            vc = rng.standard_normal(nc * Vc)
            out[f"{name}/{l}/vf"] = vf
            out[f"{name}/{l}/vc"] = vc
            out[f"{name}/{l}/restrict"] = disc.restrict(vf, l)
            out[f"{name}/{l}/prolongate"] = disc.prolongate(vc, l)
            out[f"{name}/{l}/restrict_nodal"] = disc.restrict_nodal(vf, l)
    save("transfers", **out)


def _mg_setup(name, seed):
    """Fracture level contexts like the reference's tests (test_mgsolve.py:114-136)."""
    hier = ref_hierarchy(MESHES[name])
    disc = Discretization(hier)
    space = disc.finest
    dm = space.dofmap
    rng = np.random.default_rng(seed)
    params = params_for(space, None)
    state = selfcheck.random_state(space, rng, t=0.01)
    bdry = np.unique(np.concatenate([np.nonzero(np.isclose(space.mesh.vertices[:, a], lim))[0]
                                     for a in range(hier.dim)
                                     for lim in (space.mesh.vertices[:, a].min(),
                                                 space.mesh.vertices[:, a].max())]))
    flags = np.zeros(dm.n_dofs, bool)
    for c in range(hier.dim):
        flags[dm.index(c, bdry)] = True
    vals = np.where(flags, 1e-3 * rng.standard_normal(dm.n_dofs), 0.0)
    dirichlet = ConstraintMask(flags, vals)
    active = np.zeros(dm.n_dofs, bool)
    phi_ids = np.arange(dm.phi_slice.start, dm.phi_slice.stop)
    active[phi_ids[rng.random(len(phi_ids)) < 0.2]] = True
    return disc, state, params, dirichlet, active


def gen_multigrid():
    out = {}
    for name in ("square", "lshape", "lshape3d", "cfg1"):
        t0 = time.time()
        disc, state, params, dirichlet, active = _mg_setup(name, 5)
        ctxs = mgsolve.build_level_contexts(disc, state, active, dirichlet, params,
                                            SplitKind.NOSPLIT)
        n = disc.finest.dofmap.n_dofs
        out[f"{name}/U"] = state.U
        out[f"{name}/U_prev1"] = state.U_prev1
        out[f"{name}/U_prev2"] = state.U_prev2
        out[f"{name}/phi_tilde"] = state.phi_tilde
        out[f"{name}/times"] = np.array([state.t, state.t_prev1, state.t_prev2])
        out[f"{name}/dirichlet"] = dirichlet.is_constrained
        out[f"{name}/dirichlet_vals"] = dirichlet.inhomogeneity
        out[f"{name}/active"] = active
        for l, c in enumerate(ctxs):
            out[f"{name}/{l}/diag"] = c.diag
            out[f"{name}/{l}/constrained"] = c.constrained
            out[f"{name}/{l}/spectra"] = np.array([[s.lambda_min_hat, s.lambda_max_hat, s.fallback]
                                                   for s in c.spectra], dtype=float)
        rng = np.random.default_rng(11)
        r = rng.standard_normal(n)
        out[f"{name}/r"] = r
        out[f"{name}/vcycle_full"] = mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, r)
        out[f"{name}/vcycle_full_deg3"] = mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, r,
                                                         degree=3)
        out[f"{name}/vcycle_block"] = mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.BLOCK_DIAG, r)
        fine = ctxs[-1]
        blk = fine.op.blocks[0]
        prm = mgsolve.smoother_params(fine.spectra[0], 4)
        b = rng.standard_normal(blk.stop)
        x0 = rng.standard_normal(blk.stop)
        out[f"{name}/cheb_b"] = b
        out[f"{name}/cheb_x0"] = x0
        out[f"{name}/cheb_zero"] = mgsolve.chebyshev_apply(
            lambda vb: fine.op.apply_block(0, vb), fine.diag[blk], prm, np.zeros_like(b), b)
        out[f"{name}/cheb_nonzero"] = mgsolve.chebyshev_apply(
            lambda vb: fine.op.apply_block(0, vb), fine.diag[blk], prm, x0, b)
        rc = rng.standard_normal(ctxs[0].op.n_dofs)
        out[f"{name}/coarse_r"] = rc
        out[f"{name}/coarse"] = mgsolve.coarse_solve(ctxs[0], rc)
        # one Newton-step linear solve: R~ = -A(U) with constrained rows zeroed
        mask = ctxs[-1].op.mask
        R = -model.residual(disc.finest, state, dirichlet, params, SplitKind.NOSPLIT)
        R[mask.is_constrained] = 0.0
        ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)
        x, its = krylov.gmres(fine.op.apply,
                              lambda v: mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, v),
                              R, ctl)
        out[f"{name}/gmres_rhs"] = R
        out[f"{name}/gmres_x"] = x
        out[f"{name}/gmres_iters"] = np.array(its)
        print(f"  {name}: gmres {its} iterations ({time.time() - t0:.1f}s)")
    save("multigrid", **out)


def gen_multigrid_miehe():
    """Level contexts, V-cycle and one GMRES solve with the Miehe split
    (lshape with the C^1 blend, lshape3d with the hard split)."""
    out = {}
    for name, band in (("lshape", 0.02), ("lshape3d", 0.0)):
        t0 = time.time()
        disc, state, params, dirichlet, active = _mg_setup(name, 6)
        params.split_band = band
        split = SplitKind.MIEHE
        ctxs = mgsolve.build_level_contexts(disc, state, active, dirichlet, params, split)
        n = disc.finest.dofmap.n_dofs
        out[f"{name}/band"] = np.array(band)
        out[f"{name}/U"] = state.U
        out[f"{name}/U_prev1"] = state.U_prev1
        out[f"{name}/U_prev2"] = state.U_prev2
        out[f"{name}/phi_tilde"] = state.phi_tilde
        out[f"{name}/times"] = np.array([state.t, state.t_prev1, state.t_prev2])
        out[f"{name}/dirichlet"] = dirichlet.is_constrained
        out[f"{name}/dirichlet_vals"] = dirichlet.inhomogeneity
        out[f"{name}/active"] = active
        for l, c in enumerate(ctxs):
            out[f"{name}/{l}/diag"] = c.diag
            out[f"{name}/{l}/constrained"] = c.constrained
            out[f"{name}/{l}/spectra"] = np.array([[s.lambda_min_hat, s.lambda_max_hat, s.fallback]
                                                   for s in c.spectra], dtype=float)
        rng = np.random.default_rng(12)
        r = rng.standard_normal(n)
        out[f"{name}/r"] = r
        out[f"{name}/vcycle_full"] = mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, r)
        fine = ctxs[-1]
        mask = fine.op.mask
        R = -model.residual(disc.finest, state, dirichlet, params, split)
        R[mask.is_constrained] = 0.0
        ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)
        x, its = krylov.gmres(fine.op.apply,
                              lambda v: mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, v),
                              R, ctl)
        out[f"{name}/gmres_rhs"] = R
        out[f"{name}/gmres_x"] = x
        out[f"{name}/gmres_iters"] = np.array(its)
        print(f"  {name} (miehe): gmres {its} iterations ({time.time() - t0:.1f}s)")
    save("multigrid_miehe", **out)


def _ref_problem(prob):
    hier = ref_hierarchy((prob.blocks, prob.n_levels, prob.dim))
    disc = Discretization(hier)
    st = prob.state
    state = LinearizationState(U=st.U, U_prev1=st.U_prev1, U_prev2=st.U_prev2, t=st.t,
                               t_prev1=st.t_prev1, t_prev2=st.t_prev2, phi_tilde=st.phi_tilde)
    p = prob.params
    params = MaterialParams(mu=p.mu, lam=p.lam, g_c=p.g_c, kappa=p.kappa, eps=p.eps)
    dirichlet = ConstraintMask(prob.dirichlet.is_constrained, prob.dirichlet.inhomogeneity)
    return disc, state, params, dirichlet


def gen_configs():
    from paper_1902_08112_b200 import configs
    out = {}
    for name, levels, threads, store_inputs in (("cfg1", None, 1, True), ("cfg2", 6, 8, False)):
        t0 = time.time()
        prob = configs.make(name, levels)
        tag = name if levels is None else f"{name}_l{levels}"
        disc, state, params, dirichlet = _ref_problem(prob)
        space = disc.finest
        mask = dirichlet.combined_with(prob.active, np.zeros(prob.n_dofs))
        op = model.PhaseFieldOperator(space, state, ConstraintMask(mask.is_constrained,
                                                                   mask.inhomogeneity),
                                      params, SplitKind.NOSPLIT, threads=threads)
        out[f"{tag}/checksum"] = np.array([state.U.sum(), prob.v.sum(), float(mask.is_constrained.sum())])
        if store_inputs:
            out[f"{tag}/U"] = state.U
            out[f"{tag}/v"] = prob.v
            out[f"{tag}/active"] = prob.active
            out[f"{tag}/dirichlet"] = dirichlet.is_constrained
        out[f"{tag}/apply"] = op.apply(prob.v)
        out[f"{tag}/diagonal"] = op.diagonal()
        ctxs = mgsolve.build_level_contexts(disc, state, prob.active, dirichlet, params,
                                            SplitKind.NOSPLIT, threads=threads)
        for l, c in enumerate(ctxs):
            out[f"{tag}/{l}/spectra"] = np.array([[s.lambda_min_hat, s.lambda_max_hat, s.fallback]
                                                  for s in c.spectra], dtype=float)
        R = -model.residual(space, state, dirichlet, params, SplitKind.NOSPLIT)
        R[mask.is_constrained] = 0.0
        ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)
        x, its = krylov.gmres(ctxs[-1].op.apply,
                              lambda v: mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, v,
                                                       degree=prob.degree), R, ctl)
        out[f"{tag}/gmres_rhs"] = R
        out[f"{tag}/gmres_x"] = x
        out[f"{tag}/gmres_iters"] = np.array(its)
        print(f"  {tag}: gmres {its} iterations ({time.time() - t0:.1f}s)")
    save("configs", **out)


FULL_CASES = (("cfg2", None), ("cfg4", None), ("cfg5", 6), ("cfg5", 7))
FULL_SAMPLES = 4096


def sample_index(n, seed=11):
    """Fixed sample of entries stored for full-size vectors (the whole vector
    would be tens of MB): 4096 sorted indices from default_rng(seed)."""
    return np.sort(np.random.default_rng(seed).choice(n, size=min(n, FULL_SAMPLES), replace=False))


def vec_summary(x):
    """Size-independent fingerprint of a full-size vector: 2-norm, sum, sum of
    |x|, and the entries at sample_index(n)."""
    return np.array([np.linalg.norm(x), x.sum(), np.abs(x).sum()]), x[sample_index(x.size)]


def gen_configs_full(threads=8):
    """Reference outputs at the BENCHMARKED sizes (cfg2 1024^2, cfg4 full,
    cfg5 at 96^3 = 6 levels): vmult, diagonal and Newton-residual
    fingerprints, per-level spectra, and the Newton-step GMRES iteration count
    and solution fingerprint (GMRES(30), rel 1e-8, FULL V(1,1))."""
    from paper_1902_08112_b200 import configs
    path = os.path.join(HERE, "configs_full.npz")
    out = dict(np.load(path)) if os.path.exists(path) else {}
    only = os.environ.get("FULL_ONLY")
    for name, levels in FULL_CASES:
        tag = name if levels is None else f"{name}_l{levels}"
        if only and tag not in only.split(","):
            continue
        t0 = time.time()
        prob = configs.make(name, levels)
        disc, state, params, dirichlet = _ref_problem(prob)
        space = disc.finest
        mask = dirichlet.combined_with(prob.active, np.zeros(prob.n_dofs))
        op = model.PhaseFieldOperator(space, state, ConstraintMask(mask.is_constrained,
                                                                   mask.inhomogeneity),
                                      params, SplitKind.NOSPLIT, threads=threads)
        out[f"{tag}/checksum"] = np.array([state.U.sum(), prob.v.sum(),
                                           float(mask.is_constrained.sum())])
        for key, vec in (("apply", op.apply(prob.v)), ("diagonal", op.diagonal()),
                         ("residual", model.residual(space, state, dirichlet, params,
                                                     SplitKind.NOSPLIT, threads=threads))):
            out[f"{tag}/{key}_stats"], out[f"{tag}/{key}_sample"] = vec_summary(vec)
        t1 = time.time()
        ctxs = mgsolve.build_level_contexts(disc, state, prob.active, dirichlet, params,
                                            SplitKind.NOSPLIT, threads=threads)
        t_setup = time.time() - t1
        for l, c in enumerate(ctxs):
            out[f"{tag}/{l}/spectra"] = np.array([[s.lambda_min_hat, s.lambda_max_hat, s.fallback]
                                                  for s in c.spectra], dtype=float)
        R = -model.residual(space, state, dirichlet, params, SplitKind.NOSPLIT, threads=threads)
        R[mask.is_constrained] = 0.0
        ctl = krylov.SolverControl(abs_tol=0.0, rel_tol=1e-8, restart=30, max_iters=1000)
        t1 = time.time()
        x, its = krylov.gmres(ctxs[-1].op.apply,
                              lambda v: mgsolve.vcycle(ctxs, mgsolve.PreconditionerKind.FULL, v,
                                                       degree=prob.degree), R, ctl)
        t_gmres = time.time() - t1
        out[f"{tag}/gmres_x_stats"], out[f"{tag}/gmres_x_sample"] = vec_summary(x)
        out[f"{tag}/gmres_iters"] = np.array(its)
        out[f"{tag}/ref_seconds"] = np.array([t_setup, t_gmres, float(threads)])
        print(f"  {tag}: n={prob.n_dofs} gmres {its} its, |x|={np.linalg.norm(x):.6e} "
              f"setup {t_setup:.1f}s gmres {t_gmres:.1f}s total {time.time() - t0:.1f}s", flush=True)
        np.savez_compressed(path, **out)
    print(f"  wrote configs_full.npz ({os.path.getsize(path) / 1024:.0f} KiB)")


def gen_newton(threads=8):
    """One incremental step of the reference's own Newton driver
    (nonlinear.ActiveSetSolver.solve_step, nonlinear.py:117-215), unpatched,
    on cfg1 and cfg2 at 256^2: the converged U and active set and the
    per-iteration history (set size, changed, filtered residual norm, GMRES
    iterations).  tests/test_gpu_patch.py runs the same driver with the GPU
    twins installed (patch.install) and compares."""
    from fracmg import nonlinear
    from paper_1902_08112_b200 import configs
    out = {}
    for name, levels in (("cfg1", None), ("cfg2", 6)):
        tag = name if levels is None else f"{name}_l{levels}"
        t0 = time.time()
        prob = configs.make(name, levels)
        disc, state, params, dirichlet = _ref_problem(prob)
        V = disc.finest.dofmap.n_vertices
        cfg = nonlinear.SolverConfig(cheb_degree=prob.degree, threads=threads)
        solver = nonlinear.ActiveSetSolver(disc, params, SplitKind.NOSPLIT, cfg)
        dim = disc.finest.dim
        U, rep, active = solver.solve_step(state, dirichlet, state.U[dim * V:])
        out[f"{tag}/U"] = U
        out[f"{tag}/active"] = active
        out[f"{tag}/history"] = np.array([[h.set_size, float(h.set_changed), h.residual_norm, h.gmres_iters]
                                          for h in rep.history])
        out[f"{tag}/converged"] = np.array(rep.converged)
        print(f"  {tag}: {rep.iterations} active-set iterations, gmres {rep.gmres_iters} "
              f"({time.time() - t0:.1f}s)")
    save("newton", **out)


from tests.golden.make_golden_specs import SCENARIOS, scenario  # noqa: E402


def gen_scenarios():
    """The reference's time loop scenarios.run (scenarios.py:345-426), unpatched:
    per step the active-set iterations, GMRES iterations, boundary load,
    crack and bulk energy and active-set size.  Pressurised fractures with the
    noise modulus field (NoSplit), 2D / 3D L-shapes (Miehe split with the
    run's C^1 band, LOADED boundary load)."""
    from fracmg import scenarios
    out = {}
    for tag, _, _ in SCENARIOS:
        t0 = time.time()
        recs = scenarios.run(scenario(scenarios, tag))
        out[f"{tag}/records"] = np.array([[r.step, r.time, r.active_set_iters, sum(r.gmres_iters_per_as_step),
                                           r.load, r.crack_energy, r.bulk_energy, r.n_active] for r in recs])
        print(f"  {tag}: {len(recs)} steps ({time.time() - t0:.1f}s)")
    save("scenarios", **out)


def gen_krylov():
    out = {}
    K = np.zeros((9, 9))
    for i in range(9):
        K[i, i] = 4.0
        r, c = divmod(i, 3)
        for rr, cc in ((r - 1, c), (r + 1, c), (r, c - 1), (r, c + 1)):
            if 0 <= rr < 3 and 0 <= cc < 3:
                K[i, rr * 3 + cc] = -1.0
    rng = np.random.default_rng(7)
    b = rng.standard_normal(9)
    x, its = krylov.gmres(lambda v: K @ v, None, b,
                          krylov.SolverControl(abs_tol=1e-13, rel_tol=1e-13))
    out.update(K=K, b=b, x=x, iters=np.array(its))
    n = 33
    A = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    out["lap1d"] = A
    out["lap1d_est"] = np.array([[e.lambda_min_hat, e.lambda_max_hat]
                                 for e in (krylov.estimate_spectrum(lambda v: A @ v, np.diag(A),
                                                                    n_iters=10, seed=s)
                                           for s in range(5))])
    save("krylov", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["meshes", "operator", "operator_band", "transfers", "multigrid", "multigrid_miehe", "qoi", "boundary", "configs", "newton", "scenarios", "krylov"]
    for w in which:
        print(w)
        globals()[f"gen_{w}"]()

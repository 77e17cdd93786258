"""Full-size (benchmarked) configurations: the oracle's vmult / diagonal /
Newton residual of a BASELINE config, and checks against the reference's
fingerprints in tests/golden/configs_full.npz (made by
tests/golden/make_golden.py gen_configs_full from the reference itself:
2-norm, sum, sum|.| and 4096 sampled entries of each full-size vector)."""
import os

import numpy as np

from tests.conftest import rel_err

# (config, levels, golden tag): cfg2 1024^2, cfg4 full, cfg5 at 96^3
CASES = [("cfg2", None, "cfg2"), ("cfg4", None, "cfg4"), ("cfg5", 6, "cfg5_l6")]


def sample_index(n, seed=11, k=4096):
    """The sample of make_golden.sample_index (same RNG call)."""
    return np.sort(np.random.default_rng(seed).choice(n, size=min(n, k), replace=False))


def check_fingerprint(vec, g, tag, key, tol):
    """vec (full length) against the reference's fingerprint of the same vector."""
    vec = np.asarray(vec, dtype=float)
    st = g[f"{tag}/{key}_stats"]
    assert abs(np.linalg.norm(vec) - st[0]) <= tol * st[0], (key, np.linalg.norm(vec), st[0])
    assert abs(np.abs(vec).sum() - st[2]) <= tol * st[2], key
    samp = g[f"{tag}/{key}_sample"]
    err = rel_err(vec[sample_index(vec.size)], samp)
    assert err <= tol, (key, err)
    return err


def oracle_outputs(prob, threads=None):
    """oracle/ vmult, diagonal and semilinear residual of the config (CPU)."""
    from oracle import fe, jacobian, meshgen
    threads = threads or os.cpu_count() or 1
    levels = meshgen.build_hierarchy(prob.blocks, prob.n_levels, prob.dim)
    T = fe.LevelTables(levels[-1], prob.n_levels - 1)
    p = prob.params
    mat = jacobian.Material(mu=p.mu, lam=p.lam, g_c=p.g_c, kappa=p.kappa, eps=p.eps)
    s = prob.state
    st = jacobian.State(U=s.U, U_prev1=s.U_prev1, U_prev2=s.U_prev2, t=s.t, t_prev1=s.t_prev1,
                        t_prev2=s.t_prev2, phi_tilde=s.phi_tilde)
    mask = prob.dirichlet.is_constrained | prob.active
    op = jacobian.JacobianOperator(T, st, mask, mat, threads=threads)
    out = {"apply": op.apply(prob.v), "diagonal": op.diagonal()}
    del op
    out["residual"] = jacobian.residual(T, st, prob.dirichlet.is_constrained, mat)
    return out

"""Oracle restatement of the GMG + Krylov solvers (test infrastructure).

Restates reference krylov.py (gmres 50-136, estimate_spectrum 146-198) and
mgsolve.py (Chebyshev parameters/degree 59-79, chebyshev_apply 82-113, level
contexts 128-197, blockwise smoother / coarse solve 200-218, V(1,1) cycles
221-283).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .jacobian import JacobianOperator, State


# ----------------------------------------------------------------- krylov

@dataclass
class Control:
    abs_tol: float = 1e-10
    rel_tol: float = 1e-4
    max_iters: int = 1000
    restart: int = 30


class NotConverged(RuntimeError):
    def __init__(self, x, residual_norm, iterations):
        super().__init__(f"no convergence after {iterations} iterations "
                         f"(residual {residual_norm:.3e})")
        self.x, self.residual_norm, self.iterations = x, residual_norm, iterations


def gmres(op, precond, b, control=None, x0=None):
    """Right-preconditioned restarted GMRES, MGS + conditional re-orthogonalisation,
    Givens rotations, true residual per restart (krylov.py:50-136)."""
    ctl = control or Control()
    precond = precond or (lambda v: v)
    b = np.asarray(b, dtype=float)
    x = np.zeros(b.size) if x0 is None else np.asarray(x0, dtype=float).copy()
    r = b - op(x) if x.any() else b.copy()
    rn = float(np.linalg.norm(r))
    tol = max(ctl.abs_tol, ctl.rel_tol * rn)
    if rn <= tol:
        return x, 0
    total = 0
    while True:
        m = min(ctl.restart, ctl.max_iters - total)
        if m <= 0:
            raise NotConverged(x, rn, total)
        Vb = np.zeros((m + 1, b.size))
        Zb = np.zeros((m, b.size))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        Vb[0] = r / rn
        g[0] = rn
        used = 0
        for j in range(m):
            Zb[j] = precond(Vb[j])
            w = np.array(op(Zb[j]), dtype=float)
            total += 1
            w0 = np.linalg.norm(w)
            for i in range(j + 1):
                H[i, j] = Vb[i] @ w
                w -= H[i, j] * Vb[i]
            if np.linalg.norm(w) < 1e-3 * w0:
                for i in range(j + 1):
                    c = Vb[i] @ w
                    H[i, j] += c
                    w -= c * Vb[i]
            H[j + 1, j] = np.linalg.norm(w)
            brk = H[j + 1, j] == 0.0
            if not brk:
                Vb[j + 1] = w / H[j + 1, j]
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j], H[j + 1, j] = den, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            used = j + 1
            if abs(g[j + 1]) <= tol or brk:
                break
        y = np.zeros(used)
        for i in range(used - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:used] @ y[i + 1:]) / H[i, i]
        x = x + Zb[:used].T @ y
        r = b - op(x)
        rn = float(np.linalg.norm(r))
        if rn <= tol * (1.0 + 1e-8):
            return x, total
        if total >= ctl.max_iters:
            raise NotConverged(x, rn, total)


@dataclass
class Spectrum:
    lambda_min_hat: float
    lambda_max_hat: float
    fallback: bool = False


def estimate_spectrum(op, diag, n_iters=10, seed=0, constrained=None):
    """Jacobi-PCG Lanczos extreme eigenvalues of D^-1 A (krylov.py:146-198)."""
    diag = np.asarray(diag, dtype=float)
    b = np.random.default_rng(seed).standard_normal(diag.size)
    if constrained is not None:
        b[constrained] = 0.0
    r = b.copy()
    z = r / diag
    p = z.copy()
    rz = float(r @ z)
    al, be = [], []
    for _ in range(n_iters):
        if rz <= 0.0 or not np.isfinite(rz):
            break
        Ap = op(p)
        pAp = float(p @ Ap)
        if pAp <= 0.0 or not np.isfinite(pAp):
            break
        a = rz / pAp
        al.append(a)
        r = r - a * Ap
        z = r / diag
        rz_new = float(r @ z)
        if rz_new <= 1e-28 * rz or not np.isfinite(rz_new):
            break
        be.append(rz_new / rz)
        p = z + be[-1] * p
        rz = rz_new
    k = len(al)
    if k < 2:
        return Spectrum(1.0, 1.0, True)
    T = lanczos_matrix(al, be)
    ev = np.linalg.eigvalsh(T)
    return Spectrum(float(ev[0]), float(ev[-1]), False)


def lanczos_matrix(al, be):
    """CG coefficients -> Lanczos tridiagonal (krylov.py:190-196)."""
    k = len(al)
    T = np.zeros((k, k))
    T[0, 0] = 1.0 / al[0]
    for i in range(1, k):
        T[i, i] = 1.0 / al[i] + be[i - 1] / al[i - 1]
        T[i, i - 1] = T[i - 1, i] = np.sqrt(be[i - 1]) / al[i - 1]
    return T


# ---------------------------------------------------------------- multigrid

@dataclass
class Cheb:
    degree: int
    a: float
    b: float


def smoother_range(spec, degree=4):
    """[1.2 lmax / 5, 1.2 lmax] (mgsolve.py:59-62)."""
    top = 1.2 * spec.lambda_max_hat
    return Cheb(degree, top / 5.0, top)


def solver_range(spec, degree):
    """[0.9 lmin, 1.2 lmax] (mgsolve.py:65-68)."""
    return Cheb(degree, 0.9 * spec.lambda_min_hat, 1.2 * spec.lambda_max_hat)


def solver_degree(spec, target=1e-3, cap=30):
    """mgsolve.py:71-79."""
    a, b = 0.9 * spec.lambda_min_hat, 1.2 * spec.lambda_max_hat
    if b - a <= 1e-14 * max(b, 1.0):
        return 1
    d = int(np.ceil(np.arccosh(1.0 / target) / np.arccosh((b + a) / (b - a))))
    return max(1, min(cap, d))


def chebyshev(apply_fn, diag, prm, x, b):
    """Chebyshev-accelerated Jacobi (mgsolve.py:82-113)."""
    theta = 0.5 * (prm.b + prm.a)
    delta = 0.5 * (prm.b - prm.a)
    inv = 1.0 / np.asarray(diag, dtype=float)
    x = np.asarray(x, dtype=float).copy()
    r = b - apply_fn(x) if x.any() else np.asarray(b, dtype=float).copy()
    if delta <= 1e-14 * max(abs(theta), 1.0):
        for _ in range(prm.degree):
            x += inv * r / theta
            r = b - apply_fn(x)
        return x
    sigma = theta / delta
    rho_old = 1.0 / sigma
    d = inv * r / theta
    x += d
    for _ in range(prm.degree - 1):
        r = r - apply_fn(d)
        rho = 1.0 / (2.0 * sigma - rho_old)
        d = (rho * rho_old) * d + (2.0 * rho / delta) * (inv * r)
        x += d
        rho_old = rho
    return x


@dataclass
class Level:
    level: int
    op: object
    diag: np.ndarray
    spectra: tuple
    constrained: np.ndarray
    transfers: object


def _spectra(op, diag, eig_iters, seed, level=None):
    """Seed rule seed + 31*level + 7*k (mgsolve.py:128-139)."""
    out = []
    for k, blk in enumerate(op.blocks):
        s = seed + 31 * level + 7 * k if level is not None else seed + 7 * k
        out.append(estimate_spectrum(lambda vb, k=k: op.apply_block(k, vb), diag[blk],
                                     n_iters=eig_iters, seed=s,
                                     constrained=op.constrained[blk]))
    return tuple(out)


def level_masks(transfers, fine_constrained):
    """Coarse masks = injected all-component flags (mgsolve.py:182-186)."""
    nlev = len(transfers.levels)
    nc = transfers.dim + 1
    masks = [None] * nlev
    masks[-1] = np.asarray(fine_constrained, dtype=bool)
    for l in range(nlev - 2, -1, -1):
        Vf = transfers.levels[l + 1].n_vertices
        masks[l] = masks[l + 1].reshape(nc, Vf)[:, transfers.inj[l]].ravel()
    return masks


def build_levels(transfers, tables, state, active, dirichlet_flags, material, split,
                 eig_iters=10, seed=0, threads=1):
    """mgsolve.py:154-197 (fine mask = Dirichlet | active; states by injection)."""
    nlev = len(tables)
    masks = level_masks(transfers, np.asarray(dirichlet_flags) | np.asarray(active))
    states = [None] * nlev
    states[-1] = state
    for l in range(nlev - 2, -1, -1):
        s = states[l + 1]
        states[l] = State(U=transfers.restrict_nodal(s.U, l),
                          U_prev1=transfers.restrict_nodal(s.U_prev1, l),
                          U_prev2=transfers.restrict_nodal(s.U_prev2, l),
                          t=s.t, t_prev1=s.t_prev1, t_prev2=s.t_prev2,
                          phi_tilde=transfers.inject_scalar(s.phi_tilde, l))
    out = []
    for l in range(nlev):
        op = JacobianOperator(tables[l], states[l], masks[l], material, split, threads)
        diag = op.diagonal()
        out.append(Level(l, op, diag, _spectra(op, diag, eig_iters, seed, level=l),
                         masks[l], transfers))
    return out


def _smooth(lev, x, b, degree):
    """mgsolve.py:200-206."""
    for k, blk in enumerate(lev.op.blocks):
        x[blk] = chebyshev(lambda vb, k=k: lev.op.apply_block(k, vb), lev.diag[blk],
                           smoother_range(lev.spectra[k], degree), x[blk], b[blk])
    return x


def coarse_solve(lev, r, target=1e-3, cap=30):
    """mgsolve.py:209-218."""
    x = np.zeros_like(r)
    for k, blk in enumerate(lev.op.blocks):
        prm = solver_range(lev.spectra[k], solver_degree(lev.spectra[k], target, cap))
        x[blk] = chebyshev(lambda vb, k=k: lev.op.apply_block(k, vb), lev.diag[blk],
                           prm, x[blk], r[blk])
    return x


def _cycle(levels, r, l, degree, target, cap):
    """mgsolve.py:221-235."""
    lev = levels[l]
    if l == 0:
        return coarse_solve(lev, r, target, cap)
    x = _smooth(lev, np.zeros_like(r), r, degree)
    d = r - lev.op.apply(x)
    rc = lev.transfers.restrict(d, l - 1)
    rc[levels[l - 1].constrained] = 0.0
    ec = _cycle(levels, rc, l - 1, degree, target, cap)
    ef = lev.transfers.prolongate(ec, l - 1)
    ef[lev.constrained] = 0.0
    x += ef
    return _smooth(lev, x, r, degree)


def _cycle_block(levels, k, rb, l, degree, target, cap, n_comp):
    """mgsolve.py:238-259."""
    lev = levels[l]
    blk = lev.op.blocks[k]
    ap = lambda vb: lev.op.apply_block(k, vb)  # noqa: E731
    if l == 0:
        prm = solver_range(lev.spectra[k], solver_degree(lev.spectra[k], target, cap))
        return chebyshev(ap, lev.diag[blk], prm, np.zeros_like(rb), rb)
    prm = smoother_range(lev.spectra[k], degree)
    x = chebyshev(ap, lev.diag[blk], prm, np.zeros_like(rb), rb)
    d = rb - ap(x)
    rc = lev.transfers.restrict_block(d, l - 1, n_comp)
    rc[levels[l - 1].constrained[levels[l - 1].op.blocks[k]]] = 0.0
    ec = _cycle_block(levels, k, rc, l - 1, degree, target, cap, n_comp)
    ef = lev.transfers.prolongate_block(ec, l - 1, n_comp)
    ef[lev.constrained[blk]] = 0.0
    x += ef
    return chebyshev(ap, lev.diag[blk], prm, x, rb)


def vcycle(levels, r, kind="full", degree=4, target=1e-3, cap=30):
    """mgsolve.py:262-283."""
    fine = levels[-1]
    r = np.asarray(r, dtype=float).copy()
    r[fine.constrained] = 0.0
    top = len(levels) - 1
    if kind == "full":
        return _cycle(levels, r, top, degree, target, cap)
    dim = fine.transfers.dim
    out = np.zeros_like(r)
    for k, blk in enumerate(fine.op.blocks):
        out[blk] = _cycle_block(levels, k, r[blk], top, degree, target, cap,
                                dim if k == 0 else 1)
    return out

"""Seeded synthetic inputs for the BASELINE.json configurations.

Every config is built from congruent coarse blocks exactly like the
reference's `_build_hierarchy` (mesh.py:219-222), so the vertex numbering and
level indices are the reference's.  RNG: numpy default_rng (PCG64); seed 0
for the state, 1 for the vmult vector, 2 for the fallback right-hand side.
Choices BASELINE.json leaves open follow SURVEY Appendix A.

  cfg1  2D notched unit square, 8x8 blocks, 4 levels (64^2 Q1), Cheb deg 4
  cfg2  same, 8 levels (1024^2), Cheb deg 3
  cfg4  3D L-prism [0,1]^2\\[0.5,1]^2 x [0,0.5], 0.25 blocks, 6 levels (128/unit)
  cfg5  3D unit cube, 3^3 blocks, 8 levels (384^3), penny crack r = 0.2
  cfg3  2D pressurised cracks on [-20,20]^2, 512^2 biquadratic (Q2) cells, 7 levels
        (the reference has no Q2 elements: our own Q2 definitions, oracle/q2.py)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .fem import Discretization, build_hierarchy, build_q2_hierarchy
from .model import ConstraintMask, LinearizationState, MaterialParams


@dataclass
class Problem:
    name: str
    dim: int
    blocks: list
    n_levels: int
    params: MaterialParams
    state: LinearizationState
    dirichlet: ConstraintMask
    active: np.ndarray
    v: np.ndarray
    degree: int
    disc: Discretization = None

    @property
    def n_dofs(self):
        return self.state.U.size


def tiled_blocks(counts, edge, keep=None):
    out = []
    dim = len(counts)
    for idx in np.ndindex(*tuple(counts[::-1])):
        ijk = idx[::-1]
        lo = tuple(float(i * edge) for i in ijk)
        if keep is not None and not keep(lo):
            continue
        out.append([lo, tuple(float((i + 1) * edge) for i in ijk)])
    return out


def _axes(mesh):
    """Per-vertex lattice coordinates (x, y[, z]) as float arrays, cheap for boxes."""
    if mesh.is_box:
        ext = mesh.ncell + 1
        V = int(np.prod(ext))
        idx = np.arange(V, dtype=np.int64)
        out = []
        for a in range(mesh.dim):
            out.append(((idx % ext[a]) + mesh.kmin[a]).astype(float) * mesh.cell_size[a])
            idx = idx // ext[a]
        return out
    X = mesh.vertices
    return [X[:, a] for a in range(mesh.dim)]


def _material(h):
    return MaterialParams(mu=80.77, lam=121.15, g_c=2.7e-3, kappa=1e-8, eps=2.0 * h)


def notched_square(n_levels, degree, name, stack=1):
    """cfg1/cfg2 (BASELINE configs[0], [1]).  `stack` > 1 stacks
    that many unit squares in y (weak-scaling workload: one cfg slab per GPU;
    the slit stays in the bottom square, Dirichlet rows at y = 0 and y = stack)."""
    blocks = tiled_blocks((8, 8 * stack), 1.0 / 8)
    disc = Discretization(build_hierarchy(blocks, n_levels, 2))
    mesh = disc.hierarchy.finest
    V = mesh.n_vertices
    h = float(mesh.cell_size[0])
    x, y = _axes(mesh)
    rng = np.random.default_rng(0)
    ux = rng.normal(0.0, 1e-5, V)
    uy = 1e-3 * y + rng.normal(0.0, 1e-5, V)
    phi = np.ones(V)
    slit = (np.abs(y - 0.5) < h) & (x <= 0.5)
    phi[slit] = 0.0
    U = np.concatenate([ux, uy, phi])
    flags = np.zeros(3 * V, dtype=bool)
    vals = np.zeros(3 * V)
    bottom = np.isclose(y, 0.0)
    top = np.isclose(y, float(stack))
    flags[np.nonzero(bottom)[0]] = True
    flags[V + np.nonzero(bottom)[0]] = True
    flags[np.nonzero(top)[0]] = True
    flags[V + np.nonzero(top)[0]] = True
    vals[V + np.nonzero(top)[0]] = 1e-3
    U[flags] = vals[flags]
    active = np.zeros(3 * V, dtype=bool)
    active[2 * V + np.nonzero(slit)[0]] = True
    state = LinearizationState(U=U, U_prev1=U.copy(), U_prev2=U.copy(), t=0.0, t_prev1=0.0,
                               t_prev2=0.0, phi_tilde=np.clip(phi, 0.0, 1.0))
    v = np.random.default_rng(1).standard_normal(3 * V)
    return Problem(name, 2, blocks, n_levels, _material(h), state,
                   ConstraintMask(flags, vals), active, v, degree, disc)


def lprism(n_levels=6, degree=4, name="cfg4"):
    """cfg4: 3D L-prism, 0.25 blocks (BASELINE configs[3])."""
    blocks = tiled_blocks((4, 4, 2), 0.25, keep=lambda lo: not (lo[0] >= 0.5 and lo[1] >= 0.5))
    disc = Discretization(build_hierarchy(blocks, n_levels, 3))
    mesh = disc.hierarchy.finest
    V = mesh.n_vertices
    h = float(mesh.cell_size[0])
    x, y, z = _axes(mesh)
    rng = np.random.default_rng(0)
    U = np.empty(4 * V)
    U[:3 * V] = rng.normal(0.0, 1e-5, 3 * V)
    phi = np.ones(V)
    near = np.nonzero(np.hypot(x - 0.5, y - 0.5) < 0.1)[0]
    pick = near[rng.random(near.size) < 0.05]
    phi[pick] = rng.uniform(0.0, 0.5, pick.size)
    U[3 * V:] = phi
    flags = np.zeros(4 * V, dtype=bool)
    bottom = np.nonzero(np.isclose(y, 0.0))[0]
    for c in range(3):
        flags[c * V + bottom] = True
    vals = np.zeros(4 * V)
    U[flags] = 0.0
    active = np.zeros(4 * V, dtype=bool)
    active[3 * V + pick] = True
    state = LinearizationState(U=U, U_prev1=U.copy(), U_prev2=U.copy(), t=0.0, t_prev1=0.0,
                               t_prev2=0.0, phi_tilde=np.clip(phi, 0.0, 1.0))
    v = np.random.default_rng(1).standard_normal(4 * V)
    return Problem(name, 3, blocks, n_levels, _material(h), state,
                   ConstraintMask(flags, vals), active, v, degree, disc)


def penny_cube(n_levels=8, degree=4, name="cfg5"):
    """cfg5: unit cube with a penny crack (BASELINE configs[4])."""
    blocks = tiled_blocks((3, 3, 3), 1.0 / 3)
    disc = Discretization(build_hierarchy(blocks, n_levels, 3))
    mesh = disc.hierarchy.finest
    V = mesh.n_vertices
    h = float(mesh.cell_size[0])
    eps = 2.0 * h
    x, y, z = _axes(mesh)
    rho = np.hypot(x - 0.5, y - 0.5)
    dz = z - 0.5
    d = np.where(rho <= 0.2, np.abs(dz), np.hypot(rho - 0.2, dz))
    phi = 1.0 - np.exp(-d / eps)
    disc_v = np.nonzero((np.abs(dz) < 0.25 * h) & (rho <= 0.2))[0]
    phi[disc_v] = 0.0
    rng = np.random.default_rng(0)
    U = np.empty(4 * V)
    U[:3 * V] = rng.normal(0.0, 1e-5, 3 * V)
    U[3 * V:] = phi
    flags = np.zeros(4 * V, dtype=bool)
    ends = np.nonzero(np.isclose(z, 0.0) | np.isclose(z, 1.0))[0]
    for c in range(3):
        flags[c * V + ends] = True
    vals = np.zeros(4 * V)
    U[flags] = 0.0
    active = np.zeros(4 * V, dtype=bool)
    active[3 * V + disc_v] = True
    state = LinearizationState(U=U, U_prev1=U, U_prev2=U, t=0.0, t_prev1=0.0,
                               t_prev2=0.0, phi_tilde=np.clip(phi, 0.0, 1.0))
    v = np.random.default_rng(1).standard_normal(4 * V)
    return Problem(name, 3, blocks, n_levels, _material(h), state,
                   ConstraintMask(flags, vals), active, v, degree, disc)


def _segment_distance(P, c, ang, half):
    d = np.array([np.cos(ang), np.sin(ang)])
    rel = P - c[None, :]
    t = np.clip(rel @ d, -half, half)
    return np.linalg.norm(rel - t[:, None] * d[None, :], axis=1)


def pressurized_cracks(n_levels=7, degree=4, name="cfg3", n_coarse=8):
    """cfg3 (BASELINE configs[2]): three straight phi = 0 cracks of
    length 4 with seeded centres ~ U([-15,15]^2) and angles ~ U[0, pi) in
    [-20,20]^2, biquadratic cells, p = 1e-3, u = 0 on the whole boundary,
    active set = crack nodes, u ~ N(0, 1e-4).  Material: the reference's
    fracture values (scenarios.py:223-227)."""
    disc = Discretization(build_q2_hierarchy(-20.0, 20.0, n_coarse, n_levels))
    mesh = disc.hierarchy.finest
    V = mesh.n_vertices
    h = float(mesh.cell_size[0])
    X = mesh.vertices
    rng = np.random.default_rng(0)
    centres = rng.uniform(-15.0, 15.0, (3, 2))
    angles = rng.uniform(0.0, np.pi, 3)
    crack = np.zeros(V, dtype=bool)
    for c, a in zip(centres, angles):
        crack |= _segment_distance(X, c, a, 2.0) < h
    phi = np.where(crack, 0.0, 1.0)
    U = np.empty(3 * V)
    U[:2 * V] = rng.normal(0.0, 1e-4, 2 * V)
    U[2 * V:] = phi
    bd = (np.isclose(X[:, 0], -20.0) | np.isclose(X[:, 0], 20.0) | np.isclose(X[:, 1], -20.0)
          | np.isclose(X[:, 1], 20.0))
    flags = np.zeros(3 * V, dtype=bool)
    flags[np.flatnonzero(bd)] = True
    flags[V + np.flatnonzero(bd)] = True
    U[flags] = 0.0
    active = np.zeros(3 * V, dtype=bool)
    active[2 * V + np.flatnonzero(crack)] = True
    params = MaterialParams(mu=4166.67, lam=2777.78, g_c=1.0, kappa=1e-10, eps=2.0 * h,
                            pressure_fn=lambda t: 1e-3)
    state = LinearizationState(U=U, U_prev1=U.copy(), U_prev2=U.copy(), t=0.0, t_prev1=0.0,
                               t_prev2=0.0, phi_tilde=phi.copy())
    v = np.random.default_rng(1).standard_normal(3 * V)
    return Problem(name, 2, [[(-20.0, -20.0), (20.0, 20.0)]], n_levels, params, state,
                   ConstraintMask(flags, np.zeros(3 * V)), active, v, degree, disc)


def make(name, n_levels=None):
    """Problem by config name; `n_levels` shrinks the hierarchy for parity runs."""
    if name == "cfg1":
        return notched_square(n_levels or 4, 4, name)
    if name == "cfg2":
        return notched_square(n_levels or 8, 3, name)
    if name == "cfg3":
        return pressurized_cracks(n_levels or 7, 4, name)
    if name == "cfg4":
        return lprism(n_levels or 6, 4, name)
    if name == "cfg5":
        return penny_cube(n_levels or 8, 4, name)
    raise KeyError(f"unknown config {name!r}")


def fallback_rhs(problem):
    """Seeded N(0,1) right-hand side zeroed at constrained dofs."""
    r = np.random.default_rng(2).standard_normal(problem.n_dofs)
    r[problem.dirichlet.is_constrained | problem.active] = 0.0
    return r

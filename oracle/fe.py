"""Oracle restatement of the Q1 finite-element substrate (test infrastructure).

Restates reference fem.py:
  * 2-point Gauss rule, x fastest (fem.py:33-56)
  * tensor-product Q1 values/gradients (fem.py:64-88)
  * shared per-level tables N, gradN = ref/h, JxW = w*vol (fem.py:168-188)
  * masked gather / per-component scatter (fem.py:203-225)
  * QP interpolation einsums (fem.py:229-238)
  * Q1 prolongation P (weights 1, 1/2 per axis) and vertex injection
    (fem.py:308-351) and the per-component transfers (fem.py:355-411)
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .meshgen import corner_bits, lattice_code

GAUSS_PTS = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])
GAUSS_WTS = np.array([0.5, 0.5])


def gauss_points(dim):
    """(Q, dim) points and (Q,) weights, x fastest (fem.py:44-56)."""
    bits = corner_bits(dim)                       # same enumeration as corners
    pts = GAUSS_PTS[bits]
    wts = np.prod(GAUSS_WTS[bits], axis=1)
    return pts, wts


def q1_tables(points):
    """Q1 basis values (P, n) and reference gradients (P, n, dim) (fem.py:75-88)."""
    points = np.asarray(points, dtype=float)
    npts, dim = points.shape
    bits = corner_bits(dim)
    fac = np.where(bits[None] == 1, points[:, None, :], 1.0 - points[:, None, :])
    vals = np.prod(fac, axis=2)
    grads = np.empty((npts, bits.shape[0], dim))
    sign = np.where(bits == 1, 1.0, -1.0)
    for a in range(dim):
        others = [b for b in range(dim) if b != a]
        rest = np.prod(fac[:, :, others], axis=2) if others else 1.0
        grads[:, :, a] = sign[None, :, a] * rest
    return vals, grads


class LevelTables:
    """Per-level shared tables + cells of one oracle level (fem.py:165-191)."""

    def __init__(self, level_mesh, level_index):
        self.mesh = level_mesh
        self.level = level_index
        dim = level_mesh.dim
        self.dim = dim
        self.n_comp = dim + 1
        self.n_vertices = level_mesh.n_vertices
        pts, wts = gauss_points(dim)
        vals, rgrads = q1_tables(pts)
        self.N = vals
        self.gradN = rgrads / level_mesh.cell_size[None, None, :]
        self.JxW = wts * level_mesh.cell_volume
        lo = level_mesh.vertices[level_mesh.cells[:, 0]]
        self.qp_coords = lo[:, None, :] + pts[None, :, :] * level_mesh.cell_size
        share = level_mesh.cell_volume / 2 ** dim
        self.vertex_mass = np.bincount(level_mesh.cells.ravel(),
                                       minlength=self.n_vertices) * share

    @property
    def n_dofs(self):
        return self.n_comp * self.n_vertices

    @property
    def u_slice(self):
        return slice(0, self.dim * self.n_vertices)

    @property
    def phi_slice(self):
        return slice(self.dim * self.n_vertices, self.n_dofs)

    # fem.py:203-213
    def gather(self, v, constrained=None):
        v = np.asarray(v, dtype=float)
        if constrained is not None:
            v = np.where(constrained, 0.0, v)
        comp = v.reshape(-1, self.n_vertices)
        return np.transpose(comp[:, self.mesh.cells], (1, 0, 2))

    # fem.py:215-225
    def scatter(self, local):
        ncomp = local.shape[1]
        flat = self.mesh.cells.ravel()
        parts = [np.bincount(flat, weights=np.ascontiguousarray(local[:, c]).ravel(),
                             minlength=self.n_vertices) for c in range(ncomp)]
        return np.concatenate(parts)

    # fem.py:229-238
    def at_qp(self, nodal):
        return np.einsum("cn,qn->cq", nodal, self.N)

    def grad_at_qp(self, nodal):
        return np.einsum("cn,qnj->cqj", nodal, self.gradN)

    def vec_grad_at_qp(self, nodal):
        return np.einsum("cin,qnj->cqij", nodal, self.gradN)


class Transfers:
    """Hierarchy transfers (fem.py:295-411) on oracle levels."""

    def __init__(self, levels):
        self.levels = levels
        self.dim = levels[0].dim
        self.P = [self._prolongation(l) for l in range(len(levels) - 1)]
        self.inj = [self._injection(l) for l in range(len(levels) - 1)]

    @staticmethod
    def _lookup(level):
        codes = lattice_code(level.keys, level.key_mod)
        return codes  # sorted by construction

    def _prolongation(self, l):
        """fem.py:308-344: fine key k -> coarse keys floor/ceil(k/2), weights 1 or 1/2."""
        coarse, fine = self.levels[l], self.levels[l + 1]
        kf = fine.keys
        codes_c = self._lookup(coarse)
        lo = kf // 2
        hi = (kf + 1) // 2
        odd = (kf % 2) == 1
        rows, cols, data = [], [], []
        for corner in corner_bits(self.dim):
            w = np.ones(kf.shape[0])
            key = np.where(corner[None, :] == 1, hi, lo)
            for a in range(self.dim):
                if corner[a]:
                    w *= np.where(odd[:, a], 0.5, 0.0)
                else:
                    w *= np.where(odd[:, a], 0.5, 1.0)
            keep = w > 0
            rows.append(np.nonzero(keep)[0])
            cols.append(np.searchsorted(codes_c, lattice_code(key[keep], coarse.key_mod)))
            data.append(w[keep])
        return sp.csr_matrix((np.concatenate(data),
                              (np.concatenate(rows), np.concatenate(cols))),
                             shape=(fine.n_vertices, coarse.n_vertices))

    def _injection(self, l):
        """fem.py:346-351: coarse vertex -> fine vertex with key 2k."""
        coarse, fine = self.levels[l], self.levels[l + 1]
        return np.searchsorted(self._lookup(fine),
                               lattice_code(coarse.keys * 2, fine.key_mod))

    def _per_comp(self, v, V, fn):
        return np.concatenate([fn(c) for c in np.asarray(v, dtype=float).reshape(-1, V)])

    def prolongate(self, vc, l):          # fem.py:376-383
        nc = self.dim + 1
        Vc = self.levels[l].n_vertices
        if len(vc) != nc * Vc:
            raise ValueError(f"expected {nc * Vc} dofs on level {l}, got {len(vc)}")
        return self._per_comp(vc, Vc, lambda c: self.P[l] @ c)

    def restrict(self, vf, l):            # fem.py:385-392
        nc = self.dim + 1
        Vf = self.levels[l + 1].n_vertices
        if len(vf) != nc * Vf:
            raise ValueError(f"expected {nc * Vf} dofs on level {l + 1}, got {len(vf)}")
        return self._per_comp(vf, Vf, lambda c: self.P[l].T @ c)

    def restrict_nodal(self, vf, l):      # fem.py:394-401
        Vf = self.levels[l + 1].n_vertices
        return self._per_comp(vf, Vf, lambda c: c[self.inj[l]])

    def inject_scalar(self, vf, l):       # fem.py:361-363
        return np.asarray(vf)[self.inj[l]]

    def restrict_block(self, vf, l, n_comp):    # fem.py:403-406
        Vf = self.levels[l + 1].n_vertices
        return np.concatenate([self.P[l].T @ c for c in np.asarray(vf).reshape(n_comp, Vf)])

    def prolongate_block(self, vc, l, n_comp):  # fem.py:408-411
        Vc = self.levels[l].n_vertices
        return np.concatenate([self.P[l] @ c for c in np.asarray(vc).reshape(n_comp, Vc)])

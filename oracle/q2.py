"""Oracle for biquadratic (Q2, 9-node) elements on box lattices -- test
infrastructure for BASELINE configs[2] ("512x512 Q2 quads, 3x3 Gauss points").

The reference implements Q1 only (fem.py:1-8, 33-88): there is no Q2 code to
restate, so this module extends the reference's own definitions in the
obvious way and is pinned by known-answer properties instead of golden
vectors (tests/test_oracle_q2.py): partition of unity and exact
interpolation of quadratics, exact prolongation of quadratics, rigid-body
modes in the kernel of the elasticity block, and agreement of the
sum-factorised and assembled forms.  PARITY UNPINNED (no reference output
exists for Q2).

Conventions (chosen to mirror the Q1 ones):
  * nodes = the lattice of half the cell size, x fastest (fem.py:1-4 layout
    gid = c*V + v with V = number of nodes);
  * cell nodes in lexicographic order, x fastest: local n = a + 3 b;
  * 1D Lagrange basis on {0, 1/2, 1}; 3-point Gauss rule (0.5 -/+ sqrt(3/5)/2,
    0.5; weights 5/18, 8/18, 5/18), tensor order x fastest (fem.py:44-56);
  * transfers: P = Q2 interpolation of coarse functions at fine nodes,
    R = P^T, injection coarse node i -> fine node 2i (fem.py:308-351).
The physics is the unchanged oracle/jacobian.py operator on these tables.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .fe import Transfers

G3 = np.array([0.5 - 0.5 * np.sqrt(0.6), 0.5, 0.5 + 0.5 * np.sqrt(0.6)])
W3 = np.array([5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0])


def lagrange2(t):
    """1D quadratic Lagrange basis on {0, 1/2, 1}: values (P, 3) and derivatives (P, 3)."""
    t = np.asarray(t, dtype=float)
    L = np.stack([2.0 * (t - 0.5) * (t - 1.0), -4.0 * t * (t - 1.0), 2.0 * t * (t - 0.5)], axis=-1)
    dL = np.stack([4.0 * t - 3.0, -8.0 * t + 4.0, 4.0 * t - 1.0], axis=-1)
    return L, dL


@dataclass
class Q2Level:
    """A box of nx x ny Q2 cells of size h, origin `lo` (2D)."""
    ncell: np.ndarray       # (2,) cells per axis
    cell_size: np.ndarray   # (2,)
    lo: np.ndarray          # (2,)

    dim = 2

    @property
    def n_node_axis(self):
        return 2 * self.ncell + 1

    @property
    def n_vertices(self):   # nodes (the name the Q1 code uses for its dof carriers)
        return int(np.prod(self.n_node_axis))

    @property
    def n_cells(self):
        return int(np.prod(self.ncell))

    @property
    def cell_volume(self):
        return float(np.prod(self.cell_size))

    @property
    def nodes(self):
        nxn, nyn = self.n_node_axis
        y, x = np.meshgrid(np.arange(nyn), np.arange(nxn), indexing="ij")
        return self.lo[None, :] + np.stack([x.ravel(), y.ravel()], axis=1) * (0.5 * self.cell_size)

    @property
    def cells(self):
        """(C, 9) node ids, cells x fastest, local nodes a + 3 b."""
        nx, ny = self.ncell
        nxn = 2 * nx + 1
        cy, cx = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        base = (2 * cx.ravel()) + nxn * (2 * cy.ravel())
        a = np.array([0, 1, 2] * 3)
        b = np.repeat([0, 1, 2], 3)
        return base[:, None] + a[None, :] + nxn * b[None, :]


def q2_hierarchy(lo, hi, n_coarse, n_levels):
    """Levels 0 (n_coarse^2 cells) .. n_levels-1 of the box [lo, hi]^2."""
    lo = np.asarray(lo, dtype=float) * np.ones(2)
    hi = np.asarray(hi, dtype=float) * np.ones(2)
    out = []
    for l in range(n_levels):
        n = n_coarse * 2 ** l
        out.append(Q2Level(np.array([n, n]), (hi - lo) / n, lo))
    return out


class Q2Tables:
    """The LevelTables surface (oracle/fe.py) for a Q2 level."""

    def __init__(self, level: Q2Level, level_index=0):
        self.mesh = level
        self.level = level_index
        self.dim = 2
        self.n_comp = 3
        self.n_vertices = level.n_vertices
        L, dL = lagrange2(G3)                               # (3 qp, 3 basis)
        qx = np.tile(np.arange(3), 3)                       # QP q = qx + 3 qy
        qy = np.repeat(np.arange(3), 3)
        a = np.tile(np.arange(3), 3)                        # basis n = a + 3 b
        b = np.repeat(np.arange(3), 3)
        self.N = L[qx][:, a] * L[qy][:, b]                  # (9, 9)
        h = level.cell_size
        gx = dL[qx][:, a] * L[qy][:, b] / h[0]
        gy = L[qx][:, a] * dL[qy][:, b] / h[1]
        self.gradN = np.stack([gx, gy], axis=-1)            # (9, 9, 2)
        self.JxW = W3[qx] * W3[qy] * level.cell_volume
        pts = np.stack([G3[qx], G3[qy]], axis=1)
        nx, ny = level.ncell
        cy, cx = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        cell_lo = level.lo[None, :] + np.stack([cx.ravel(), cy.ravel()], axis=1) * h
        self.qp_coords = cell_lo[:, None, :] + pts[None, :, :] * h
        self._cells = level.cells

    @property
    def n_dofs(self):
        return self.n_comp * self.n_vertices

    @property
    def u_slice(self):
        return slice(0, self.dim * self.n_vertices)

    @property
    def phi_slice(self):
        return slice(self.dim * self.n_vertices, self.n_dofs)

    def gather(self, v, constrained=None):
        v = np.asarray(v, dtype=float)
        if constrained is not None:
            v = np.where(constrained, 0.0, v)
        comp = v.reshape(-1, self.n_vertices)
        return np.transpose(comp[:, self._cells], (1, 0, 2))

    def scatter(self, local):
        ncomp = local.shape[1]
        flat = self._cells.ravel()
        parts = [np.bincount(flat, weights=np.ascontiguousarray(local[:, c]).ravel(),
                             minlength=self.n_vertices) for c in range(ncomp)]
        return np.concatenate(parts)

    def at_qp(self, nodal):
        return np.einsum("cn,qn->cq", nodal, self.N)

    def grad_at_qp(self, nodal):
        return np.einsum("cn,qnj->cqj", nodal, self.gradN)

    def vec_grad_at_qp(self, nodal):
        return np.einsum("cin,qnj->cqij", nodal, self.gradN)


def _prolongation_1d(nc_cells):
    """(2*(2nc)+1) x (2nc+1) Q2 interpolation of one axis (fine nodes x coarse nodes)."""
    nfn = 4 * nc_cells + 1
    ncn = 2 * nc_cells + 1
    rows, cols, vals = [], [], []
    for j in range(nfn):
        if j % 2 == 0:
            rows.append(j)
            cols.append(j // 2)
            vals.append(1.0)
            continue
        c = j // 4
        t = (j - 4 * c) / 4.0
        L, _ = lagrange2(np.array([t]))
        for k in range(3):
            rows.append(j)
            cols.append(2 * c + k)
            vals.append(float(L[0, k]))
    return sp.csr_matrix((vals, (rows, cols)), shape=(nfn, ncn))


class Q2Transfers(Transfers):
    """P (Q2 interpolation, tensor product of the 1D operators) and node injection."""

    def __init__(self, levels):
        self.levels = levels
        self.dim = 2
        self.P = []
        self.inj = []
        for l in range(len(levels) - 1):
            c = levels[l]
            px = _prolongation_1d(int(c.ncell[0]))
            py = _prolongation_1d(int(c.ncell[1]))
            P = sp.kron(py, px).tocsr()                     # x fastest
            P.eliminate_zeros()
            self.P.append(P)
            nxc, nyc = c.n_node_axis
            nxf = 2 * nxc - 1
            iy, ix = np.meshgrid(np.arange(nyc), np.arange(nxc), indexing="ij")
            self.inj.append((2 * ix.ravel() + nxf * 2 * iy.ravel()).astype(np.int64))

"""Lattice description of a level mesh and its device-side descriptor.

The reference meshes (mesh.py:163-222) are unions of congruent axis-aligned
blocks refined uniformly; vertex ids are lattice points sorted with x fastest
(mesh.py:48-52, 176-178).  For a box domain the id of lattice point (x, y, z)
is x + (nx+1)(y + (ny+1) z); for a non-box union (the L-shapes) every row of
constant (y, z) is a contiguous run of ids, described by per-row tables.

`LatticeMesh` / `build_hierarchy` build that numbering natively (no key
sorting; arrays that only the reference needs -- keys, cells, vertices -- are
produced lazily).  `lattice_of(mesh)` accepts either a `LatticeMesh` or any
reference `LevelMesh` (keys + cells arrays) and returns the device
descriptor used by every kernel.
"""
from __future__ import annotations

import ctypes as C
from functools import cached_property

import numpy as np
import torch

from . import _lib


def corner_bits(dim):
    idx = np.arange(2 ** dim)
    return np.stack([(idx >> a) & 1 for a in range(dim)], axis=1).astype(np.int64)


class LatticeMesh:
    """One refined level of a block union, lattice-native.

    Exposes the reference LevelMesh attributes used on the hot path
    (dim, n_vertices, n_cells, cell_size, cell_volume, diameter, keys,
    key_mod, vertices, cells) -- the array ones lazily.
    """

    def __init__(self, blocks, level, dim, tagger=None):
        self.tagger = tagger                                     # mesh.py:196-206 (None: all OUTER)
        blocks = np.asarray(blocks, dtype=float).reshape(-1, 2, dim)
        n = 2 ** level
        spacing = (blocks[0, 1] - blocks[0, 0]) / n
        self.dim = dim
        self.level_refinement = n
        self.cell_size = np.asarray(spacing, dtype=float)
        self.key_mod = int(round((blocks[:, 1] / spacing).max())) + 2
        lows = np.rint(blocks[:, 0] / spacing).astype(np.int64)
        self.kmin = lows.min(axis=0)
        rel = lows - self.kmin
        self.block_lows = rel                                    # (B, dim) in cells
        self.ncell = (rel + n).max(axis=0)                       # cells per axis of the bbox
        self.is_box = int(len(blocks)) * n ** dim == int(np.prod(self.ncell))
        if not self.is_box:
            self._build_rows()

    # -- occupancy / row tables (non-box only) ------------------------------
    def _occupancy(self, vertices):
        n = self.level_refinement
        ext = self.ncell + (1 if vertices else 0)
        occ = np.zeros(tuple(ext[::-1]), dtype=bool)               # (z, y, x) / (y, x)
        span = n + 1 if vertices else n
        for lo in self.block_lows:
            sl = tuple(slice(lo[a], lo[a] + span) for a in range(self.dim))[::-1]
            occ[sl] = True
        return occ

    def _build_rows(self):
        vocc = self._occupancy(True).reshape(-1, self.ncell[0] + 1)
        cocc = self._occupancy(False).reshape(-1, self.ncell[0])
        self.vrow_lo, self.vrow_hi, cnt = _row_runs(vocc)
        self.vrow_off = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64)
        self.crow_lo, self.crow_hi, ccnt = _row_runs(cocc)
        self._nv = int(cnt.sum())
        self._nc = int(ccnt.sum())

    # -- LevelMesh surface ----------------------------------------------------
    @property
    def n_vertices(self):
        if self.is_box:
            return int(np.prod(self.ncell + 1))
        return self._nv

    @property
    def n_cells(self):
        if self.is_box:
            return int(np.prod(self.ncell))
        return self._nc

    @property
    def cell_volume(self):
        return float(np.prod(self.cell_size))

    @property
    def diameter(self):
        return float(np.linalg.norm(self.cell_size))

    @cached_property
    def keys(self):
        if self.is_box:
            grids = np.meshgrid(*[np.arange(e + 1) for e in self.ncell[::-1]], indexing="ij")
            rel = np.stack([g.ravel() for g in grids[::-1]], axis=1)
        else:
            rel = np.argwhere(self._occupancy(True))[:, ::-1]
        return (rel + self.kmin).astype(np.int64)

    @cached_property
    def vertices(self):
        return self.keys.astype(float) * self.cell_size

    def vertex_ids(self, rel):
        """Ids of lattice points rel (..., dim) relative to kmin (-1 if absent)."""
        rel = np.asarray(rel, dtype=np.int64)
        x = rel[..., 0]
        nxv, nyv = self.ncell[0] + 1, self.ncell[1] + 1
        row = rel[..., 1] + (nyv * rel[..., 2] if self.dim == 3 else 0)
        if self.is_box:
            return x + nxv * row
        lo, hi = self.vrow_lo[row], self.vrow_hi[row]
        ids = self.vrow_off[row] + (x - lo)
        return np.where((x >= lo) & (x < hi), ids, -1)

    @cached_property
    def cell_coords(self):
        """Lattice coordinates (relative to kmin) of every cell, in mesh cell
        order: block by block, x fastest inside a block (mesh.py:180-194)."""
        n = self.level_refinement
        grids = np.meshgrid(*([np.arange(n)] * self.dim), indexing="ij")
        local = np.stack([g.ravel() for g in grids[::-1]], axis=1)
        return (self.block_lows[:, None, :] + local[None, :, :]).reshape(-1, self.dim)

    @cached_property
    def cells(self):
        """Cells block by block, x fastest inside a block, corners x fastest
        (mesh.py:180-194)."""
        corners = self.cell_coords[:, None, :] + corner_bits(self.dim)[None, :, :]
        return self.vertex_ids(corners)

    def lattice_cell_index(self, cell_ids):
        """Lattice cell index cx + nx (cy + ny cz) of mesh cells."""
        c = self.cell_coords[np.asarray(cell_ids, dtype=np.int64)]
        idx = c[:, -1]
        for a in range(self.dim - 2, -1, -1):
            idx = idx * self.ncell[a] + c[:, a]
        return idx.astype(np.int64)

    # -- boundary faces (mesh.py:149-161, 196-206) -----------------------------
    @cached_property
    def _boundary(self):
        occ = self._occupancy(False)                     # (z, y, x) / (y, x) cell occupancy
        c = self.cell_coords
        nf = 2 * self.dim
        bnd = np.zeros((c.shape[0], nf), dtype=bool)
        for f in range(nf):
            a, side = f // 2, f % 2
            nb = c.copy()
            nb[:, a] += 1 if side else -1
            inside = (nb[:, a] >= 0) & (nb[:, a] < self.ncell[a])
            nbc = np.clip(nb, 0, self.ncell - 1)
            exists = occ[tuple(nbc[:, ::-1].T)] & inside
            bnd[:, f] = ~exists
        rows = np.nonzero(bnd.ravel())[0]                # cell-major, face-minor: the reference order
        bf_cell, bf_face = rows // nf, rows % nf
        lo = (c[bf_cell] + self.kmin).astype(float) * self.cell_size
        hi = (c[bf_cell] + self.kmin + 1).astype(float) * self.cell_size
        axis, side = bf_face // 2, bf_face % 2
        k = np.arange(len(bf_face))
        plane = (c[bf_cell, axis] + self.kmin[axis] + side).astype(float) * self.cell_size[axis]
        lo[k, axis] = plane
        hi[k, axis] = plane
        if self.tagger is None:
            tag = np.zeros(len(bf_cell), dtype=np.int64)
        else:
            tag = np.asarray(self.tagger(lo, hi, axis, side), dtype=np.int64)
        return bf_cell.astype(np.int64), bf_face.astype(np.int64), tag

    @property
    def bf_cell(self):
        return self._boundary[0]

    @property
    def bf_face(self):
        return self._boundary[1]

    @property
    def bf_tag(self):
        return self._boundary[2]

    def cell_lower_corners(self, cell_ids):
        """Coordinates of the low corner of mesh cells (LevelMesh.cell_bounds()[0])."""
        c = self.cell_coords[np.asarray(cell_ids, dtype=np.int64)]
        return (c + self.kmin).astype(float) * self.cell_size


def _row_runs(occ):
    """Per-row [lo, hi) of a boolean (rows, width) array; each row must be one run."""
    width = occ.shape[1]
    cnt = occ.sum(axis=1)
    has = cnt > 0
    lo = np.where(has, np.argmax(occ, axis=1), 0)
    hi = np.where(has, width - np.argmax(occ[:, ::-1], axis=1), 0)
    if np.any(hi - lo != cnt):
        raise NotImplementedError("lattice rows with gaps are not supported "
                                  "(every row of constant (y, z) must be one run)")
    return lo.astype(np.int32), hi.astype(np.int32), cnt.astype(np.int64)


def build_hierarchy(blocks, n_levels, dim, tagger=None):
    """Levels 0 (coarsest) .. n_levels-1 of a block union (mesh.py:219-222);
    `tagger(fv_lo, fv_hi, axis, side)` tags the boundary faces as there."""
    return [LatticeMesh(blocks, l, dim, tagger) for l in range(n_levels)]


class Q2LatticeMesh:
    """A 2D box of nx x ny biquadratic (Q2, 9-node) cells (BASELINE configs[2]).

    The reference has Q1 elements only; Q2 dofs live on the nodes of the
    half-spacing lattice, numbered x fastest like the Q1 vertices
    (oracle/q2.py holds the matching CPU definitions).  `n_vertices` is the
    node count (the component stride of every dof vector)."""

    order = 2
    dim = 2
    is_box = True

    def __init__(self, lo, hi, ncell):
        self.lo = np.asarray(lo, dtype=float) * np.ones(2)
        hi = np.asarray(hi, dtype=float) * np.ones(2)
        self.ncell = np.asarray(ncell, dtype=np.int64) * np.ones(2, dtype=np.int64)
        self.cell_size = (hi - self.lo) / self.ncell
        info = LatticeInfo(2, self.ncell, self.cell_size, self.n_vertices, True)
        info.order = 2
        self.lattice_info = info

    @property
    def n_node_axis(self):
        return 2 * self.ncell + 1

    @property
    def n_vertices(self):
        return int(np.prod(self.n_node_axis))

    @property
    def n_cells(self):
        return int(np.prod(self.ncell))

    @property
    def cell_volume(self):
        return float(np.prod(self.cell_size))

    @property
    def diameter(self):
        return float(np.linalg.norm(self.cell_size))

    @cached_property
    def vertices(self):
        """Node coordinates (V, 2), x fastest."""
        nxn, nyn = self.n_node_axis
        y, x = np.meshgrid(np.arange(nyn), np.arange(nxn), indexing="ij")
        return self.lo[None, :] + np.stack([x.ravel(), y.ravel()], axis=1) * (0.5 * self.cell_size)

    @cached_property
    def cells(self):
        """(C, 9) node ids, cells x fastest, local nodes a + 3 b."""
        nx, ny = (int(v) for v in self.ncell)
        nxn = 2 * nx + 1
        cy, cx = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        base = 2 * cx.ravel() + nxn * 2 * cy.ravel()
        a = np.array([0, 1, 2] * 3)
        b = np.repeat([0, 1, 2], 3)
        return base[:, None] + a[None, :] + nxn * b[None, :]


def build_q2_hierarchy(lo, hi, n_coarse, n_levels):
    """Q2 levels 0 (n_coarse^2 cells) .. n_levels-1 of the box [lo, hi]^2."""
    return [Q2LatticeMesh(lo, hi, n_coarse * 2 ** l) for l in range(n_levels)]


# --------------------------------------------------------------- descriptors

class LatticeInfo:
    """Host-side lattice facts of any level mesh (ours or the reference's)."""

    def __init__(self, dim, ncell, h, n_vertices, is_box, rows=None, cell_perm=None):
        self.dim = dim
        self.ncell = np.asarray(ncell, dtype=np.int64)
        self.h = np.asarray(h, dtype=float)
        self.n_vertices = int(n_vertices)
        self.is_box = is_box
        self.rows = rows                 # (vrow_off, vrow_lo, vrow_hi, crow_lo, crow_hi) or None
        self.cell_perm = cell_perm       # mesh cell index -> lattice cell index (for rho)
        self.own = (0, 0)                # finalised planes of the last axis; (0, 0) = all
        self.order = 1                   # element order (2: Q2 node lattice)

    @property
    def n_planes(self):
        """Planes of the last axis: vertex planes (Q1) or node rows (Q2)."""
        return (2 if getattr(self, "order", 1) == 2 else 1) * int(self.ncell[-1]) + 1

    def plane_offsets(self):
        """Vertex id of the first vertex of every plane of the last axis (+ V)."""
        if getattr(self, "order", 1) == 2:
            nxn, nyn = 2 * self.ncell + 1
            return np.arange(nyn + 1, dtype=np.int64) * nxn
        if self.rows is None:
            per = int(np.prod(self.ncell[:-1] + 1))
            return np.arange(self.n_planes + 1, dtype=np.int64) * per
        voff, vlo, vhi = self.rows[0], self.rows[1], self.rows[2]
        rows_per_plane = int(self.ncell[1]) + 1 if self.dim == 3 else 1
        counts = (np.asarray(vhi, np.int64) - np.asarray(vlo, np.int64)).reshape(self.n_planes, -1).sum(1)
        return np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)

    def slab(self, lo, hi, own):
        """Sub-lattice of vertex planes [lo, hi] (inclusive) with the finalised
        planes `own` = (own_lo, own_hi) given in global plane numbers."""
        offs = self.plane_offsets()
        ncell = self.ncell.copy()
        q2 = getattr(self, "order", 1) == 2
        if q2:                             # planes are node rows; a slab is whole cell layers
            assert lo % 2 == 0 and hi % 2 == 0, (lo, hi)
        ncell[-1] = (hi - lo) // 2 if q2 else hi - lo
        rows = None
        if self.rows is not None:
            voff, vlo, vhi, clo, chi = self.rows
            rpp = int(self.ncell[1]) + 1 if self.dim == 3 else 1           # vertex rows per plane
            cpp = int(self.ncell[1]) if self.dim == 3 else 1                # cell rows per plane
            vs = slice(lo * rpp, (hi + 1) * rpp)
            cs = slice(lo * cpp, hi * cpp)
            rows = (np.asarray(voff[vs], np.int64) - offs[lo], vlo[vs], vhi[vs], clo[cs], chi[cs])
        out = LatticeInfo(self.dim, ncell, self.h, int(offs[hi + 1] - offs[lo]), self.is_box, rows)
        out.own = (own[0] - lo, own[1] - lo)
        out.order = 2 if q2 else 1
        out.global_offset = int(offs[lo])
        out.plane_lo = int(lo)
        return out


def info_from_mesh(mesh):
    if hasattr(mesh, "lattice_info"):
        return mesh.lattice_info
    if isinstance(mesh, LatticeMesh):
        rows = None if mesh.is_box else (mesh.vrow_off, mesh.vrow_lo, mesh.vrow_hi,
                                         mesh.crow_lo, mesh.crow_hi)
        return LatticeInfo(mesh.dim, mesh.ncell, mesh.cell_size, mesh.n_vertices, mesh.is_box, rows)
    return _info_from_arrays(mesh)


def _info_from_arrays(mesh):
    """Derive the lattice of a reference LevelMesh from its keys and cells and
    verify that the numbering is the lattice numbering the kernels assume."""
    keys = np.asarray(mesh.keys, dtype=np.int64)
    cells = np.asarray(mesh.cells, dtype=np.int64)
    dim = keys.shape[1]
    kmin = keys.min(axis=0)
    rel = keys - kmin
    ncell = rel.max(axis=0)
    nxv = int(ncell[0]) + 1
    nrows = int(ncell[1] + 1) * (int(ncell[2] + 1) if dim == 3 else 1)
    row = rel[:, 1] + ((ncell[1] + 1) * rel[:, 2] if dim == 3 else 0)
    V = keys.shape[0]
    if np.any(np.diff(row) < 0):
        raise ValueError("mesh vertices are not in lattice order (x fastest)")
    is_box = V == nxv * nrows
    rows = None
    if is_box:
        ids = rel[:, 0] + nxv * row
        if not np.array_equal(ids, np.arange(V)):
            raise ValueError("box mesh vertex numbering is not the lattice numbering")
    else:
        vocc = np.zeros((nrows, nxv), dtype=bool)
        vocc[row, rel[:, 0]] = True
        vlo, vhi, cnt = _row_runs(vocc)
        voff = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64)
        ids = voff[row] + rel[:, 0] - vlo[row]
        if not np.array_equal(ids, np.arange(V)):
            raise ValueError("mesh vertex numbering is not row-contiguous lattice order")
    # cells: corner 0 gives the lattice cell; verify all corners
    c0 = rel[cells[:, 0]]
    bits = corner_bits(dim)
    for n in range(2 ** dim):
        if not np.array_equal(rel[cells[:, n]], c0 + bits[n]):
            raise ValueError("mesh cells are not lattice cells with x-fastest corners")
    ncx, ncy = int(ncell[0]), int(ncell[1])
    crow = c0[:, 1] + (ncy * c0[:, 2] if dim == 3 else 0)
    cell_perm = c0[:, 0] + ncx * crow
    ncrows = ncy * (int(ncell[2]) if dim == 3 else 1)
    cocc = np.zeros((ncrows, ncx), dtype=bool)
    cocc[crow, c0[:, 0]] = True
    if cocc.sum() != cells.shape[0]:
        raise ValueError("duplicate cells in mesh")
    if not is_box or cells.shape[0] != ncx * ncrows:
        if is_box:
            raise ValueError("box vertex set with missing cells is not supported")
        clo, chi, _ = _row_runs(cocc)
        rows = (voff, vlo, vhi, clo, chi)
    return LatticeInfo(dim, ncell, mesh.cell_size, V, is_box, rows, cell_perm)


TILE3 = 15      # PFFMG_TILE3 (include/pffmg.h): vertex columns per 3D streaming-kernel tile edge


def occupied_tiles3d(info):
    """pffmg_lattice.tiles3d of a 3D non-box lattice: the ascending indices
    bx + ntx*by of the TILE3 x TILE3 vertex-column tiles that hold a vertex
    (None for 2D and box lattices, whose tiles are all occupied)."""
    if info.dim != 3 or info.rows is None:
        return None
    _, vlo, vhi, _, _ = info.rows
    nxv, nyv = int(info.ncell[0]) + 1, int(info.ncell[1]) + 1
    ntx, nty = -(-nxv // TILE3), -(-nyv // TILE3)
    vlo = np.asarray(vlo).reshape(-1, nyv)          # rows r = y + (ny+1) z
    vhi = np.asarray(vhi).reshape(-1, nyv)
    occ = np.zeros((nty, ntx), dtype=bool)
    for bx in range(ntx):
        lo, hi = bx * TILE3, min((bx + 1) * TILE3, nxv)
        hit = ((vhi > vlo) & (vlo < hi) & (vhi > lo)).any(axis=0)     # per vertex row y
        for by in range(nty):
            occ[by, bx] = hit[by * TILE3:(by + 1) * TILE3].any()
    return np.flatnonzero(occ.ravel()).astype(np.int32)


class DeviceLattice:
    """pffmg_lattice + the device row tables backing it."""

    def __init__(self, info: LatticeInfo):
        self.info = info
        self.dim = info.dim
        self.n_vertices = info.n_vertices
        L = _lib.Lattice()
        L.dim = info.dim
        L.nx, L.ny = int(info.ncell[0]), int(info.ncell[1])
        L.nz = int(info.ncell[2]) if info.dim == 3 else 0
        L.hx, L.hy = float(info.h[0]), float(info.h[1])
        L.hz = float(info.h[2]) if info.dim == 3 else 0.0
        L.n_vertices = info.n_vertices
        self._tables = []
        if info.rows is not None:
            dev = torch.device("cuda")
            voff, vlo, vhi, clo, chi = info.rows
            ts = [torch.as_tensor(np.ascontiguousarray(voff, dtype=np.int64), device=dev),
                  torch.as_tensor(np.ascontiguousarray(vlo, dtype=np.int32), device=dev),
                  torch.as_tensor(np.ascontiguousarray(vhi, dtype=np.int32), device=dev),
                  torch.as_tensor(np.ascontiguousarray(clo, dtype=np.int32), device=dev),
                  torch.as_tensor(np.ascontiguousarray(chi, dtype=np.int32), device=dev)]
            self._tables = ts
            L.vrow_off, L.vrow_lo, L.vrow_hi, L.crow_lo, L.crow_hi = [t.data_ptr() for t in ts]
        L.own_lo, L.own_hi = int(info.own[0]), int(info.own[1])
        L.plane0 = int(getattr(info, "plane_lo", 0))
        L.order = int(getattr(info, "order", 1))
        tiles = occupied_tiles3d(info)
        if tiles is not None:
            t = torch.as_tensor(tiles, device="cuda")
            self._tables.append(t)
            L.tiles3d, L.n_tiles3d = t.data_ptr(), int(t.numel())
        self.struct = L
        self.ref = C.byref(L)
        self._rows = {}
        # host plane offsets for pffmg_apply_host (NULL = box numbering)
        self.plane_off_host = (None if info.rows is None
                               else np.ascontiguousarray(info.plane_offsets(), dtype=np.int64))

    def rows(self, lo, hi):
        """The same lattice finalising only planes [lo, hi) of the last axis."""
        key = (int(lo), int(hi))
        ref = self._rows.get(key)
        if ref is None:
            L = _lib.Lattice()
            C.pointer(L)[0] = self.struct
            L.own_lo, L.own_hi = key
            ref = self._rows[key] = (L, C.byref(L))
        return ref[1]

    @property
    def n_lattice_cells(self):
        return int(np.prod(self.info.ncell))


_CACHE = {}


def device_lattice(mesh):
    """Cached DeviceLattice of a mesh object (ours or the reference's)."""
    key = id(mesh)
    hit = _CACHE.get(key)
    if hit is not None and hit[0] is mesh:
        return hit[1]
    _lib.require_cuda()
    dl = DeviceLattice(info_from_mesh(mesh))
    _CACHE[key] = (mesh, dl)
    return dl

"""Oracle restatement of the nested block-lattice hierarchy (test infrastructure).

Restates reference mesh.py:163-222 (`_build_level`, `_build_hierarchy`):
a level is the union of congruent axis-aligned blocks, each refined into
2**level cells per axis.  Vertices are unique integer lattice keys sorted by
the linear code sum_a key[a] * mod**a (so x runs fastest, mesh.py:48-52);
cells are listed block by block, x fastest inside a block, corners in
lexicographic order with x fastest (mesh.py:36-39, 180-194).

Boundary-face tagging (mesh.py:149-160, 196-205) is not on the hot path and
is not restated.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def corner_bits(dim):
    """(2**dim, dim) 0/1 offsets, x fastest (mesh.py:36-39)."""
    idx = np.arange(2 ** dim)
    return np.stack([(idx >> a) & 1 for a in range(dim)], axis=1).astype(np.int64)


def lattice_code(keys, mod):
    """Linear code of integer keys, x least significant (mesh.py:48-52)."""
    keys = np.asarray(keys, dtype=np.int64)
    code = np.zeros(keys.shape[0], dtype=np.int64)
    mult = 1
    for a in range(keys.shape[1]):
        code += keys[:, a] * mult
        mult *= mod
    return code


@dataclass
class OracleLevel:
    vertices: np.ndarray   # (V, dim)
    cells: np.ndarray      # (C, 2**dim)
    cell_size: np.ndarray  # (dim,)
    keys: np.ndarray       # (V, dim) int64
    key_mod: int

    @property
    def dim(self):
        return self.vertices.shape[1]

    @property
    def n_vertices(self):
        return self.vertices.shape[0]

    @property
    def n_cells(self):
        return self.cells.shape[0]

    @property
    def cell_volume(self):
        return float(np.prod(self.cell_size))

    @property
    def diameter(self):
        return float(np.linalg.norm(self.cell_size))


def build_level(blocks, level, dim):
    """One refined level of a block union (mesh.py:163-216)."""
    blocks = np.asarray(blocks, dtype=float)
    n = 2 ** level
    spacing = (blocks[0, 1] - blocks[0, 0]) / n
    mod = int(round((blocks[:, 1] / spacing).max())) + 2
    lows = np.rint(blocks[:, 0] / spacing).astype(np.int64)      # (B, dim)

    # every block contributes an (n+1)^dim patch of lattice keys
    local = np.stack(np.meshgrid(*([np.arange(n + 1)] * dim), indexing="ij"),
                     axis=-1).reshape(-1, dim)[:, ::-1]          # x fastest
    all_keys = (lows[:, None, :] + local[None, :, :]).reshape(-1, dim)
    codes = np.unique(lattice_code(all_keys, mod))
    keys = np.empty((codes.size, dim), dtype=np.int64)
    rest = codes.copy()
    for a in range(dim):
        keys[:, a] = rest % mod
        rest //= mod

    cell_local = np.stack(np.meshgrid(*([np.arange(n)] * dim), indexing="ij"),
                          axis=-1).reshape(-1, dim)[:, ::-1]     # x fastest
    bits = corner_bits(dim)
    corner_keys = (lows[:, None, None, :] + cell_local[None, :, None, :]
                   + bits[None, None, :, :])                     # (B, n^d, 2^d, d)
    corner_codes = lattice_code(corner_keys.reshape(-1, dim), mod)
    cells = np.searchsorted(codes, corner_codes).reshape(-1, 2 ** dim)
    return OracleLevel(vertices=keys.astype(float) * spacing, cells=cells,
                       cell_size=np.asarray(spacing, dtype=float), keys=keys,
                       key_mod=mod)


def build_hierarchy(blocks, n_levels, dim):
    """Levels 0 (coarsest) .. n_levels-1 (mesh.py:219-222)."""
    return [build_level(blocks, l, dim) for l in range(n_levels)]


def square_blocks(side, dim=2):
    """Single-block square/cube (mesh.py:225-236)."""
    return [[(0.0,) * dim, (float(side),) * dim]]


def lshape_blocks(side, extrude=None):
    """Three-block L-shape, lower-right quadrant removed (mesh.py:239-265)."""
    s = float(side)
    b = s / 2.0
    b2 = [[(0.0, 0.0), (b, b)], [(0.0, b), (b, s)], [(b, b), (s, s)]]
    if extrude is None:
        return b2
    return [[lo + (0.0,), hi + (float(extrude),)] for lo, hi in b2]


def tiled_blocks(counts, edge, dim, keep=None):
    """A grid of congruent blocks of edge `edge`, `counts` per axis, optionally
    filtered by keep(lo) -> bool (used for the BASELINE configs)."""
    out = []
    for idx in np.ndindex(*tuple(counts[::-1])):
        ijk = idx[::-1]
        lo = tuple(float(i * edge) for i in ijk)
        if keep is not None and not keep(lo):
            continue
        hi = tuple(float((i + 1) * edge) for i in ijk)
        out.append([lo, hi])
    return out

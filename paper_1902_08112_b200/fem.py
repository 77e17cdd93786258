"""Drop-in twin of the reference level/transfer surface (fem.py) on sm_100a kernels.

`Discretization(hierarchy)` exposes the transfer API of reference
fem.py:295-411 -- prolongate / restrict / restrict_nodal / inject_scalar /
injection / restrict_block / prolongate_block / *_scalar -- implemented as
lattice stencil kernels (libpffmg pffmg_restrict / pffmg_prolongate /
pffmg_inject_*) instead of scipy CSR products.  It accepts our lattice
hierarchy (`build_hierarchy`) or a reference GridHierarchy, and numpy or CUDA
vectors (results have the input's kind).  Size checks raise ValueError with
the reference's messages (fem.py:380-400).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .arrays import dev, empty, host, like
from .lattice import LatticeMesh, build_hierarchy as _build_levels, device_lattice

__all__ = ["DofMap", "LevelSpace", "Hierarchy", "Discretization", "build_hierarchy", "build_q2_hierarchy"]


class DofMap:
    """Component-major dof numbering gid = c*V + v (reference fem.py:91-126)."""

    def __init__(self, mesh):
        self.mesh = mesh
        self.n_vertices = mesh.n_vertices
        self.dim = mesh.dim
        self.n_components = mesh.dim + 1

    @property
    def n_dofs(self):
        return self.n_components * self.n_vertices

    def index(self, component, vertex):
        return component * self.n_vertices + np.asarray(vertex)

    @property
    def u_slice(self):
        return slice(0, self.dim * self.n_vertices)

    @property
    def phi_slice(self):
        return slice(self.dim * self.n_vertices, self.n_dofs)


class LevelSpace:
    """Minimal level bundle for lattice meshes (reference fem.py:165-199)."""

    def __init__(self, mesh, level):
        self.mesh = mesh
        self.level = level
        self.dofmap = DofMap(mesh)

    @property
    def n_dofs(self):
        return self.dofmap.n_dofs

    @property
    def dim(self):
        return self.mesh.dim

    @property
    def vertex_mass(self):
        """Gauss-Lobatto lumped mass (fem.py:184-188)."""
        share = self.mesh.cell_volume / 2 ** self.dim
        return np.bincount(np.asarray(self.mesh.cells).ravel(),
                           minlength=self.mesh.n_vertices).astype(float) * share


@dataclass
class Hierarchy:
    """Levels coarse -> fine (reference mesh.py:125-146)."""
    dim: int
    levels: list

    @property
    def n_levels(self):
        return len(self.levels)

    @property
    def finest(self):
        return self.levels[-1]


def build_hierarchy(blocks, n_levels, dim, tagger=None):
    """Lattice-native twin of mesh._build_hierarchy (mesh.py:219-222)."""
    return Hierarchy(dim, _build_levels(blocks, n_levels, dim, tagger))


def build_q2_hierarchy(lo, hi, n_coarse, n_levels):
    """Biquadratic (Q2) box hierarchy (BASELINE configs[2]; no reference counterpart)."""
    from .lattice import build_q2_hierarchy as _q2
    return Hierarchy(2, _q2(lo, hi, n_coarse, n_levels))


class Discretization:
    """Hierarchy-wide bundle: spaces + device transfers (fem.py:295-411)."""

    def __init__(self, hierarchy, spaces=None):
        self.hierarchy = hierarchy
        self.spaces = spaces if spaces is not None else [
            LevelSpace(m, l) for l, m in enumerate(hierarchy.levels)]
        self._inj = {}

    @classmethod
    def wrap(cls, disc):
        """Our transfers over a reference Discretization's own levels/spaces."""
        if isinstance(disc, Discretization):
            return disc
        return cls(disc.hierarchy, disc.spaces)

    @property
    def finest(self):
        return self.spaces[-1]

    @property
    def dim(self):
        return self.hierarchy.dim

    def lattice(self, l):
        return device_lattice(self.hierarchy.levels[l])

    def _pair(self, l):
        return self.lattice(l), self.lattice(l + 1)

    # -- device-level kernels ------------------------------------------------
    def restrict_dev(self, vf, vc, l, n_comp, comp0=0, coarse_flags=None):
        c, f = self._pair(l)
        _lib.call("pffmg_restrict", c.ref, f.ref, n_comp, comp0, _lib.ptr(vf), _lib.ptr(vc),
                  _lib.ptr(coarse_flags), _lib.stream())

    def restrict_init_bd_dev(self, vf, vc, l, coarse_flags, inv, theta_u, theta_p, r, d, x):
        """restrict_dev of all components fused with the coarse level's
        block-diagonal Chebyshev start from x = 0 (pffmg_restrict_init_bd)."""
        c, f = self._pair(l)
        _lib.call("pffmg_restrict_init_bd", c.ref, f.ref, _lib.ptr(vf), _lib.ptr(vc), _lib.ptr(coarse_flags),
                  _lib.ptr(inv), _lib.ptr(theta_u), _lib.ptr(theta_p), _lib.ptr(r), _lib.ptr(d), _lib.ptr(x),
                  _lib.stream())

    def prolongate_dev(self, vc, vf, l, n_comp, comp0=0, fine_flags=None, accumulate=False):
        c, f = self._pair(l)
        _lib.call("pffmg_prolongate", c.ref, f.ref, n_comp, comp0, _lib.ptr(vc), _lib.ptr(vf),
                  _lib.ptr(fine_flags), int(accumulate), _lib.stream())

    def inject_dev(self, vf, vc, l, n_comp):
        c, f = self._pair(l)
        _lib.call("pffmg_inject_f64", c.ref, f.ref, n_comp, _lib.ptr(vf), _lib.ptr(vc), _lib.stream())

    def inject_flags_dev(self, ff, fc, l):
        c, f = self._pair(l)
        _lib.call("pffmg_inject_flags", c.ref, f.ref, _lib.ptr(ff), _lib.ptr(fc), _lib.stream())

    # -- reference surface ---------------------------------------------------
    def _V(self, l):
        return self.hierarchy.levels[l].n_vertices

    def _check(self, v, l, n_comp, what):
        if len(v) != n_comp * self._V(l):
            raise ValueError(f"expected {n_comp * self._V(l)} dofs on level {l}, got {len(v)}")

    def _prol(self, v_coarse, l, n_comp):
        x = dev(v_coarse)
        out = empty(n_comp * self._V(l + 1))
        self.prolongate_dev(x, out, l, n_comp)
        return like(out, v_coarse)

    def _rest(self, v_fine, l, n_comp):
        x = dev(v_fine)
        out = empty(n_comp * self._V(l))
        self.restrict_dev(x, out, l, n_comp)
        return like(out, v_fine)

    def _inj_vec(self, v_fine, l, n_comp):
        x = dev(v_fine)
        out = empty(n_comp * self._V(l))
        self.inject_dev(x, out, l, n_comp)
        return like(out, v_fine)

    def prolongate_scalar(self, v, l):
        return self._prol(v, l, 1)

    def restrict_scalar(self, v, l):
        return self._rest(v, l, 1)

    def inject_scalar(self, v, l):
        return self._inj_vec(v, l, 1)

    def injection(self, l):
        """Coarse vertex id -> coincident fine vertex id (fem.py:346-351), int64 numpy."""
        if l not in self._inj:
            c, f = self._pair(l)
            out = torch.empty(self._V(l), dtype=torch.int64, device="cuda")
            _lib.call("pffmg_injection_map", c.ref, f.ref, _lib.ptr(out), _lib.stream())
            self._inj[l] = host(out)
        return self._inj[l]

    def prolongate(self, v_coarse, l):
        nc = self.dim + 1
        if len(v_coarse) != nc * self._V(l):
            raise ValueError(f"expected {nc * self._V(l)} dofs on level {l}, got {len(v_coarse)}")
        return self._prol(v_coarse, l, nc)

    def restrict(self, v_fine, l):
        nc = self.dim + 1
        if len(v_fine) != nc * self._V(l + 1):
            raise ValueError(f"expected {nc * self._V(l + 1)} dofs on level {l + 1}, got {len(v_fine)}")
        return self._rest(v_fine, l, nc)

    def restrict_nodal(self, v_fine, l):
        nc = self.dim + 1
        if len(v_fine) != nc * self._V(l + 1):
            raise ValueError(f"expected {nc * self._V(l + 1)} dofs on level {l + 1}, got {len(v_fine)}")
        return self._inj_vec(v_fine, l, nc)

    def restrict_block(self, v_fine, l, n_comp):
        return self._rest(v_fine, l, n_comp)

    def prolongate_block(self, v_coarse, l, n_comp):
        return self._prol(v_coarse, l, n_comp)

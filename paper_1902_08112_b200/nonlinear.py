"""GPU twins of the active-set helpers of reference nonlinear.py.

`lumped_mass_inverse(space)` (nonlinear.py:67-72) and
`compute_active_set(R, U, phi_old, mass_inv, params, dofmap, dirichlet_flags)`
(nonlinear.py:75-89) with the reference's signatures.  The classification
runs in one kernel (libpffmg `pffmg_active_set`) with the reference's
rounding, so the set is bit-exact for identical inputs; the reference's
Newton driver itself (ActiveSetSolver) is the caller and stays on the host.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .arrays import dev, empty, host, is_tensor, like, pack_flags
from .lattice import info_from_mesh

__all__ = ["lumped_mass_inverse", "compute_active_set"]


def _vertex_mass(space):
    """Gauss-Lobatto lumped mass: (#adjacent cells) * vol / 2^d (fem.py:184-188)."""
    mesh = space.mesh
    share = float(np.prod(mesh.cell_size)) / 2 ** mesh.dim
    cells = getattr(mesh, "cells", None)
    return np.bincount(np.asarray(cells).ravel(), minlength=mesh.n_vertices).astype(float) * share


def lumped_mass_inverse(space):
    """Reciprocal lumped mass, one entry per dof (nonlinear.py:67-72)."""
    m = getattr(space, "vertex_mass", None)
    m = _vertex_mass(space) if m is None else np.asarray(m)
    if np.any(m <= 0.0):
        raise RuntimeError("lumped mass has non-positive entries")
    nc = space.mesh.dim + 1 if hasattr(space.mesh, "dim") else space.dofmap.n_components
    return np.tile(1.0 / m, nc)


def compute_active_set(R, U, phi_old, mass_inv, params, dofmap, dirichlet_flags=None):
    """Phase-field dofs where phi <= phi_old is enforced (nonlinear.py:75-89)."""
    _lib.require_cuda()
    V = dofmap.n_vertices
    nc = dofmap.n_components
    d = nc - 1
    Rd, Ud, Md = dev(R), dev(U), dev(mass_inv)
    po = dev(phi_old)
    flags = None
    if dirichlet_flags is not None:
        flags = pack_flags(dirichlet_flags, nc, V)
    act = torch.zeros(nc * V, dtype=torch.uint8, device="cuda")
    _lib.call("pffmg_active_set", _lib.ptr(Rd[d * V:]), _lib.ptr(Ud[d * V:]), _lib.ptr(po),
              _lib.ptr(Md[d * V:]), float(params.c), _lib.ptr(flags), d, V, _lib.ptr(act[d * V:]),
              _lib.stream())
    out = act.to(torch.bool)
    return like(out, R)

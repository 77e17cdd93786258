"""Shared specs of the golden cases (imported by make_golden.py and the tests).

Meshes are given as (blocks, n_levels, dim) -- the arguments of the
reference's `_build_hierarchy` (mesh.py:219-222); the reference's own test
meshes (tests/conftest.py:7-19) plus small versions of the BASELINE configs.
"""
import numpy as np


def _tiled(counts, edge, keep=None):
    out = []
    for idx in np.ndindex(*tuple(counts[::-1])):
        ijk = idx[::-1]
        lo = tuple(float(i * edge) for i in ijk)
        if keep is not None and not keep(lo):
            continue
        out.append([lo, tuple(float((i + 1) * edge) for i in ijk)])
    return out


def _lshape(s, extrude=None):
    b = s / 2.0
    b2 = [[(0.0, 0.0), (b, b)], [(0.0, b), (b, s)], [(b, b), (s, s)]]
    if extrude is None:
        return b2
    return [[lo + (0.0,), hi + (float(extrude),)] for lo, hi in b2]


MESHES = {
    # reference test meshes: build_square(4.0, 3), build_lshape(500, 2[, extrude=250])
    "square": ([[(0.0, 0.0), (4.0, 4.0)]], 3, 2),
    "lshape": (_lshape(500.0), 2, 2),
    "lshape3d": (_lshape(500.0, 250.0), 2, 3),
    # BASELINE config geometries at small size
    "cfg1": (_tiled((8, 8), 1.0 / 8), 4, 2),
    "cube": (_tiled((3, 3, 3), 1.0 / 3), 2, 3),
    "lprism": (_tiled((4, 4, 2), 0.25, keep=lambda lo: not (lo[0] >= 0.5 and lo[1] >= 0.5)), 2, 3),
    "rect3d": ([[(0.0, 0.0, 0.0), (2.0, 1.0, 0.5)]], 3, 3),
}


def modulus(X):
    """A smooth positive modulus field rho(x) (MaterialParams.modulus_field)."""
    X = np.asarray(X, dtype=float)
    return 1.0 + 0.3 * np.sin(0.9 * X[..., 0] + 0.2) + 0.2 * np.cos(0.7 * X[..., 1])


def params_for(space, modulus_field=None, cls=None):
    """Reference selfcheck parameters (selfcheck.py:161-165), eps scaled to the mesh."""
    if cls is None:
        from fracmg.model import MaterialParams as cls  # noqa: N813
    scale = 1.0 if space.mesh.cell_size[0] < 10 else 250.0
    return cls(mu=1.3, lam=0.9, g_c=0.7, kappa=1e-10, eps=2.0 * scale,
               pressure_fn=lambda t: 10.0 * t, modulus_field=modulus_field)


def face_tagger(fv_lo, fv_hi, axis, side):
    """Boundary tags of the boundary-load goldens (mesh.py:196-206 tagger
    signature): y-low faces FIXED (1), y-high LOADED (2), x faces
    TRACTION_FREE (3), the rest OUTER (0)."""
    axis = np.asarray(axis)
    side = np.asarray(side)
    tag = np.zeros(len(axis), dtype=np.int64)
    tag[axis == 0] = 3
    tag[(axis == 1) & (side == 0)] = 1
    tag[(axis == 1) & (side == 1)] = 2
    return tag

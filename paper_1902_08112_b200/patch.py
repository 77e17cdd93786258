"""Drop-in installation into an imported reference `fracmg`.

The reference's Newton driver resolves its hot-path entry points through
module attributes at call time (`mgsolve.build_level_contexts`,
`mgsolve.vcycle`, `krylov.gmres`; reference nonlinear.py:170-181).  `install`
points those attributes (and the other hot-path functions of mgsolve/krylov)
at the GPU twins; `uninstall` restores the originals.

    import fracmg
    from paper_1902_08112_b200 import patch
    patch.install(fracmg)                  # ActiveSetSolver now runs on the GPU
"""
from __future__ import annotations

import importlib

_SAVED = {}

MGSOLVE = ["build_level_contexts", "contexts_from_operators", "vcycle", "coarse_solve",
           "chebyshev_apply"]
KRYLOV = ["gmres", "estimate_spectrum"]


MODEL_PHYSICS = ["residual", "crack_energy", "bulk_energy", "fracture_volume", "boundary_load"]
NONLINEAR = ["compute_active_set"]


def install(fracmg=None, operator=False, physics=False):
    """Swap the GPU twins into `fracmg` (module or None to import it).

    operator=True also replaces `fracmg.model.PhaseFieldOperator` (NoSplit
    and the Miehe split, 2D and 3D).  physics=True also replaces the Newton
    right-hand side `model.residual`, the QoIs `model.crack_energy /
    bulk_energy / fracture_volume / boundary_load` and `nonlinear.compute_active_set`, which
    the reference's ActiveSetSolver and scenarios.run look up at call time
    (nonlinear.py:146-150, 195; scenarios.py:411-415)."""
    if fracmg is None:
        fracmg = importlib.import_module("fracmg")
    from . import krylov, mgsolve, model
    ref_mg = importlib.import_module(fracmg.__name__ + ".mgsolve")
    ref_kr = importlib.import_module(fracmg.__name__ + ".krylov")
    ref_model = importlib.import_module(fracmg.__name__ + ".model")
    for name in MGSOLVE:
        _SAVED.setdefault((ref_mg, name), getattr(ref_mg, name))
        setattr(ref_mg, name, getattr(mgsolve, name))
    for name in KRYLOV:
        _SAVED.setdefault((ref_kr, name), getattr(ref_kr, name))
        setattr(ref_kr, name, getattr(krylov, name))
    # the reference's `except krylov.NoConvergence` must catch our raise
    krylov._NO_CONVERGENCE[0] = ref_kr.NoConvergence
    if operator:
        _SAVED.setdefault((ref_model, "PhaseFieldOperator"), ref_model.PhaseFieldOperator)
        ref_model.PhaseFieldOperator = model.PhaseFieldOperator
    if physics:
        from . import nonlinear
        ref_nl = importlib.import_module(fracmg.__name__ + ".nonlinear")
        for name in MODEL_PHYSICS:
            _SAVED.setdefault((ref_model, name), getattr(ref_model, name))
            setattr(ref_model, name, getattr(model, name))
        for name in NONLINEAR:
            _SAVED.setdefault((ref_nl, name), getattr(ref_nl, name))
            setattr(ref_nl, name, getattr(nonlinear, name))
    return fracmg


def uninstall():
    from . import krylov
    for (mod, name), fn in list(_SAVED.items()):
        setattr(mod, name, fn)
    _SAVED.clear()
    krylov._NO_CONVERGENCE[0] = krylov.NoConvergence


def installed():
    return bool(_SAVED)

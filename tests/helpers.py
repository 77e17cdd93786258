"""Builders shared by the tests: oracle objects and product objects from the
golden specs (tests/golden/specs.py)."""
import numpy as np

from oracle import fe, jacobian, meshgen, solvers
from tests.golden.specs import MESHES, modulus, params_for


def oracle_levels(name):
    blocks, n_levels, dim = MESHES[name]
    return meshgen.build_hierarchy(blocks, n_levels, dim)


def oracle_stack(name):
    levels = oracle_levels(name)
    tables = [fe.LevelTables(m, l) for l, m in enumerate(levels)]
    return levels, tables, fe.Transfers(levels)


def oracle_material(tables, with_modulus=False):
    return params_for(tables, modulus if with_modulus else None, cls=jacobian.Material)


def oracle_state(U, phi_tilde, t):
    return jacobian.State(U=U, U_prev1=U, U_prev2=U, t=float(t), t_prev1=0.0, t_prev2=0.0,
                          phi_tilde=phi_tilde)


def product_disc(name):
    from paper_1902_08112_b200.fem import Discretization, build_hierarchy
    blocks, n_levels, dim = MESHES[name]
    return Discretization(build_hierarchy(blocks, n_levels, dim))


def product_params(space, with_modulus=False):
    from paper_1902_08112_b200.model import MaterialParams
    return params_for(space, modulus if with_modulus else None, cls=MaterialParams)


def product_state(U, phi_tilde, t, U_prev1=None, U_prev2=None, t_prev1=0.0, t_prev2=0.0):
    from paper_1902_08112_b200.model import LinearizationState
    return LinearizationState(U=U, U_prev1=U if U_prev1 is None else U_prev1,
                              U_prev2=U if U_prev2 is None else U_prev2, t=float(t),
                              t_prev1=float(t_prev1), t_prev2=float(t_prev2), phi_tilde=phi_tilde)


OP_TAGS = [(m, v) for m in MESHES for v in ("plain", "masked", "modulus")]

import sys, os, numpy as np
sys.path.insert(0, "/root/reference/pkg/src"); sys.path.insert(0, "/root/repo")
from fracmg import fem, nonlinear
from tests.golden.make_golden import ref_hierarchy, save
from tests.golden.specs import MESHES
out = {}
rng = np.random.default_rng(42)
for name in ("square", "lshape3d", "cfg1"):
    disc = fem.Discretization(ref_hierarchy(MESHES[name]))
    space = disc.finest
    dm = space.dofmap
    minv = nonlinear.lumped_mass_inverse(space)
    out[f"{name}/mass_inv"] = minv
    for k in range(3):
        R = rng.standard_normal(dm.n_dofs) * (100 if k == 0 else 1)
        U = rng.standard_normal(dm.n_dofs)
        po = rng.standard_normal(dm.n_vertices)
        dflags = rng.random(dm.n_dofs) < 0.2
        act = nonlinear.compute_active_set(R, U, po, minv, nonlinear.ActiveSetParams(c=100.0), dm,
                                           dirichlet_flags=dflags if k == 2 else None)
        for key, val in dict(R=R, U=U, phi_old=po, dflags=dflags, active=act).items():
            out[f"{name}/{k}/{key}"] = val
save("nonlinear", **out)

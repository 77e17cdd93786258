"""A numpy Laplace + reaction level operator implementing the reference's
block protocol (the shape of reference tests/modelproblem.py:13-132), used to
exercise the generic (non-native) multigrid path.  Test infrastructure."""
import numpy as np

from oracle import fe


class Mask:
    def __init__(self, flags):
        self.is_constrained = flags
        self.inhomogeneity = np.zeros(flags.size)


class LaplaceReaction:
    def __init__(self, mesh, level, flags, eps):
        self.space = fe.LevelTables(mesh, level)
        self.mask = Mask(flags)
        self.eps = eps

    @property
    def blocks(self):
        return (self.space.u_slice, self.space.phi_slice)

    def _u(self, lu):
        T = self.space
        g = np.einsum("cin,qnj->cqij", lu, T.gradN)
        return np.einsum("q,cqij,qnj->cin", T.JxW, g, T.gradN)

    def _p(self, lp):
        T = self.space
        out = np.einsum("q,cq,qn->cn", T.JxW, T.at_qp(lp), T.N) / self.eps
        out += self.eps * np.einsum("q,cqj,qnj->cn", T.JxW, T.grad_at_qp(lp), T.gradN)
        return out

    def apply(self, v):
        v = np.asarray(v, dtype=float)
        T = self.space
        loc = T.gather(v, self.mask.is_constrained)
        out = T.scatter(np.concatenate([self._u(loc[:, :T.dim]), self._p(loc[:, T.dim])[:, None]], 1))
        c = self.mask.is_constrained
        out[c] = v[c]
        return out

    def apply_block(self, k, vb):
        vb = np.asarray(vb, dtype=float)
        T = self.space
        c = self.mask.is_constrained[self.blocks[k]]
        vz = np.where(c, 0.0, vb)
        cells = T.mesh.cells
        if k == 0:
            loc = np.transpose(vz.reshape(T.dim, T.n_vertices)[:, cells], (1, 0, 2))
            out = T.scatter(self._u(loc))
        else:
            out = T.scatter(self._p(vz[cells])[:, None])
        out[c] = vb[c]
        return out

    def diagonal(self):
        T = self.space
        g2 = np.einsum("q,qnj,qnj->n", T.JxW, T.gradN, T.gradN)
        n2 = np.einsum("q,qn,qn->n", T.JxW, T.N, T.N)
        C = T.mesh.n_cells
        local = np.empty((C, T.dim + 1, T.N.shape[1]))
        local[:, :T.dim] = g2
        local[:, T.dim] = n2 / self.eps + self.eps * g2
        out = T.scatter(local)
        out[self.mask.is_constrained] = 1.0
        return out


def build_model_problem(disc, eps):
    hier = disc.hierarchy
    dim = hier.dim
    nc = dim + 1
    fine = hier.levels[-1]
    X = fine.vertices
    bd = np.zeros(fine.n_vertices, bool)
    for a in range(dim):
        bd |= np.isclose(X[:, a], X[:, a].min()) | np.isclose(X[:, a], X[:, a].max())
    flags = np.zeros(nc * fine.n_vertices, bool)
    for c in range(dim):
        flags[c * fine.n_vertices + np.nonzero(bd)[0]] = True
    masks = [None] * hier.n_levels
    masks[-1] = flags
    for l in range(hier.n_levels - 2, -1, -1):
        Vf = hier.levels[l + 1].n_vertices
        masks[l] = masks[l + 1].reshape(nc, Vf)[:, disc.injection(l)].ravel()
    return [LaplaceReaction(hier.levels[l], l, masks[l], eps) for l in range(hier.n_levels)]

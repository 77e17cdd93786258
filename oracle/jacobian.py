"""Oracle restatement of the linearised phase-field Jacobian (test infrastructure).

Restates reference model.py:
  * MaterialParams / LinearizationState fields (model.py:89-119)
  * extrapolate, degradation (model.py:122-141)
  * NoSplit and Miehe (spectral, C^1-blended) strain splits (model.py:65-86, 148-219)
  * PhaseFieldOperator caches (model.py:270-309), _lin_stress (313-323),
    block and full local kernels (325-355), chunked threading (237-239, 357-364),
    apply / apply_block / diagonal (368-413)
  * residual (model.py:420-460) -- the Newton right-hand side
  * quantities of interest crack_energy, bulk_energy, fracture_volume (model.py:472-504)
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, replace
from typing import Callable, Optional

import numpy as np

NOSPLIT = "none"
MIEHE = "miehe"
EIG_GAP_TOL = 1e-8     # model.py:48


@dataclass
class Material:
    mu: float
    lam: float
    g_c: float
    kappa: float = 1e-10
    eps: float = 1.0
    pressure_fn: Optional[Callable[[float], float]] = None
    modulus_field: Optional[Callable[[np.ndarray], np.ndarray]] = None
    split_band: float = 0.0

    def pressure(self, t):
        return float(self.pressure_fn(t)) if self.pressure_fn is not None else 0.0


@dataclass
class State:
    U: np.ndarray
    U_prev1: np.ndarray
    U_prev2: np.ndarray
    t: float
    t_prev1: float
    t_prev2: float
    phi_tilde: np.ndarray

    def with_U(self, U):
        return replace(self, U=U)


def extrapolate(p1, p2, t, t1, t2):
    """model.py:122-132."""
    p1 = np.asarray(p1, dtype=float)
    if t1 - t2 <= 0.0:
        return np.clip(p1, 0.0, 1.0)
    return np.clip(p1 + (t - t1) * (p1 - np.asarray(p2, dtype=float)) / (t1 - t2), 0.0, 1.0)


def degradation(phi, kappa):
    """model.py:135-137."""
    return (1.0 - kappa) * np.square(phi) + kappa


def _pos(x, band):
    if band <= 0.0:
        return np.maximum(x, 0.0)
    return np.where(x >= band, x, np.where(x <= -band, 0.0, np.square(x + band) / (4.0 * band)))


def _pos_prime(x, band):
    if band <= 0.0:
        return (x > 0.0).astype(float)
    return np.where(x >= band, 1.0, np.where(x <= -band, 0.0, (x + band) / (2.0 * band)))


def _pos_sq(x, band):
    if band <= 0.0:
        return np.square(np.maximum(x, 0.0))
    return np.where(x >= band, np.square(x) + band ** 2 / 3.0,
                    np.where(x <= -band, 0.0, (x + band) ** 3 / (6.0 * band)))


def split_quantities(e, kind, lam, mu, need_tangent=False, band=0.0):
    """E+, E-, sigma+, sigma-, dsigma+ of symmetric strains e (..., d, d) (model.py:148-219)."""
    d = e.shape[-1]
    eye = np.eye(d)
    tr = np.trace(e, axis1=-2, axis2=-1)
    if kind == NOSPLIT:
        Ep = 0.5 * lam * tr ** 2 + mu * np.einsum("...ij,...ij->...", e, e)
        sp = 2.0 * mu * e + lam * tr[..., None, None] * eye
        return Ep, np.zeros_like(Ep), sp, np.zeros_like(sp), None
    w, vec = np.linalg.eigh(e)
    scale = np.linalg.norm(e, axis=(-2, -1))
    wp = _pos(w, band)
    trp = _pos(tr, band)
    Es = 0.5 * lam * tr ** 2 + mu * np.sum(w ** 2, axis=-1)
    Ep = 0.5 * lam * _pos_sq(tr, band) + mu * np.sum(_pos_sq(w, band), axis=-1)
    ep = np.einsum("...ia,...a,...ja->...ij", vec, wp, vec)
    sig = 2.0 * mu * e + lam * tr[..., None, None] * eye
    sp = 2.0 * mu * ep + lam * trp[..., None, None] * eye
    tangent = None
    if need_tangent:
        H = _pos_prime(w, band)
        P4 = np.zeros(e.shape + (d, d))
        for a in range(d):
            M = np.einsum("...i,...j->...ij", vec[..., :, a], vec[..., :, a])
            P4 += H[..., a, None, None, None, None] * np.einsum("...ij,...kl->...ijkl", M, M)
        for a in range(d):
            for b in range(a + 1, d):
                gap = w[..., a] - w[..., b]
                degen = np.abs(gap) < EIG_GAP_TOL * np.maximum(scale, 1e-300)
                dd = np.where(degen, 0.5 * (H[..., a] + H[..., b]),
                              (wp[..., a] - wp[..., b]) / np.where(degen, 1.0, gap))
                S = 0.5 * (np.einsum("...i,...j->...ij", vec[..., :, a], vec[..., :, b])
                           + np.einsum("...i,...j->...ij", vec[..., :, b], vec[..., :, a]))
                P4 += 2.0 * dd[..., None, None, None, None] * np.einsum("...ij,...kl->...ijkl", S, S)
        Htr = _pos_prime(tr, band)
        tangent = lam * Htr[..., None, None, None, None] * np.einsum("ij,kl->ijkl", eye, eye) \
            + 2.0 * mu * P4
    return Ep, Es - Ep, sp, sig - sp, tangent


def _chunks(n, threads):
    b = np.linspace(0, n, threads + 1).astype(int)
    return [(b[i], b[i + 1]) for i in range(threads) if b[i + 1] > b[i]]


class JacobianOperator:
    """Matrix-free constrained Jacobian of one level (model.py:242-413)."""

    def __init__(self, tables, state, constrained, material, split=NOSPLIT, threads=1):
        self.space = tables
        self.state = state
        self.constrained = np.asarray(constrained, dtype=bool)
        self.material = material
        self.split = split
        self.threads = max(1, int(threads))
        self._pool = None
        self._cache()

    @property
    def blocks(self):
        return (self.space.u_slice, self.space.phi_slice)

    def _cache(self):
        """model.py:270-309."""
        sp_, m, dim = self.space, self.material, self.space.dim
        loc = sp_.gather(self.state.U)
        gu = sp_.vec_grad_at_qp(loc[:, :dim])
        eu = 0.5 * (gu + np.swapaxes(gu, -1, -2))
        div = np.trace(gu, axis1=-2, axis2=-1)
        phi_q = sp_.at_qp(loc[:, dim])
        gk = degradation(sp_.at_qp(np.asarray(self.state.phi_tilde)[sp_.mesh.cells]), m.kappa)
        rho = (np.asarray(m.modulus_field(sp_.qp_coords), dtype=float)
               if m.modulus_field is not None else np.ones_like(phi_q))
        p = m.pressure(self.state.t)
        Ep, _, sp, _, tangent = split_quantities(eu, self.split, m.lam, m.mu,
                                                 need_tangent=self.split == MIEHE,
                                                 band=m.split_band)
        self.rho = rho
        self.gk_rho = gk * rho
        self.gkm1_rho = (gk - 1.0) * rho
        self.tangent = tangent
        self.T = (rho[..., None, None] * (1.0 - m.kappa) * phi_q[..., None, None] * sp
                  + 2.0 * p * phi_q[..., None, None] * np.eye(dim))
        self.a = (1.0 - m.kappa) * rho * Ep + 2.0 * p * div + m.g_c / m.eps
        self.k_phi = m.g_c * m.eps

    def _stress(self, e, rows):
        """model.py:313-323."""
        m = self.material
        tr = np.trace(e, axis1=-2, axis2=-1)
        iso = 2.0 * m.mu * e + m.lam * tr[..., None, None] * np.eye(self.space.dim)
        if self.split == NOSPLIT:
            return self.gk_rho[rows, :, None, None] * iso
        extra = np.einsum("cqijkl,cqkl->cqij", self.tangent[rows], e)
        return self.rho[rows, :, None, None] * iso + self.gkm1_rho[rows, :, None, None] * extra

    def _loc_u(self, lu, rows):
        sp_ = self.space
        g = sp_.vec_grad_at_qp(lu)
        s = self._stress(0.5 * (g + np.swapaxes(g, -1, -2)), rows)
        return np.einsum("q,cqij,qnj->cin", sp_.JxW, s, sp_.gradN)

    def _loc_phi(self, lp, rows):
        sp_ = self.space
        out = np.einsum("q,cq,qn->cn", sp_.JxW, self.a[rows] * sp_.at_qp(lp), sp_.N)
        out += self.k_phi * np.einsum("q,cqj,qnj->cn", sp_.JxW, sp_.grad_at_qp(lp), sp_.gradN)
        return out

    def _loc_full(self, loc, rows):
        """model.py:340-355."""
        sp_, dim = self.space, self.space.dim
        out = np.empty_like(loc)
        g = sp_.vec_grad_at_qp(loc[:, :dim])
        s = self._stress(0.5 * (g + np.swapaxes(g, -1, -2)), rows)
        out[:, :dim] = np.einsum("q,cqij,qnj->cin", sp_.JxW, s, sp_.gradN)
        val = sp_.at_qp(loc[:, dim])
        vphi = np.einsum("cqij,cqij->cq", self.T[rows], g) + self.a[rows] * val
        out[:, dim] = np.einsum("q,cq,qn->cn", sp_.JxW, vphi, sp_.N)
        out[:, dim] += self.k_phi * np.einsum("q,cqj,qnj->cn", sp_.JxW,
                                              sp_.grad_at_qp(loc[:, dim]), sp_.gradN)
        return out

    def _run(self, kernel, loc):
        """Chunked threading, results concatenated in order (model.py:357-364)."""
        if self.threads == 1 or loc.shape[0] < 2 * self.threads:
            return kernel(loc, slice(None))
        if self._pool is None:
            self._pool = ThreadPoolExecutor(max_workers=self.threads)
        futs = [self._pool.submit(kernel, loc[a:b], slice(a, b))
                for a, b in _chunks(loc.shape[0], self.threads)]
        return np.concatenate([f.result() for f in futs], axis=0)

    def apply(self, v):
        """model.py:368-375."""
        v = np.asarray(v, dtype=float)
        out = self.space.scatter(self._run(self._loc_full,
                                           self.space.gather(v, self.constrained)))
        out[self.constrained] = v[self.constrained]
        return out

    def apply_block(self, which, vb):
        """model.py:377-392."""
        vb = np.asarray(vb, dtype=float)
        dim, V = self.space.dim, self.space.n_vertices
        c = self.constrained[self.blocks[which]]
        vz = np.where(c, 0.0, vb)
        cells = self.space.mesh.cells
        if which == 0:
            loc = np.transpose(vz.reshape(dim, V)[:, cells], (1, 0, 2))
            local = self._run(self._loc_u, loc)
        else:
            loc = vz[cells]
            local = self._run(self._loc_phi, loc)[:, None, :]
        out = self.space.scatter(local)
        out[c] = vb[c]
        return out

    def diagonal(self):
        """model.py:394-413 with the single-basis strain tables of fem.py:242-261."""
        sp_, m, dim = self.space, self.material, self.space.dim
        G = sp_.gradN                                        # (Q, n, d)
        Q, n = G.shape[0], G.shape[1]
        esym = np.zeros((dim, n, Q, dim, dim))
        for i in range(dim):
            for a in range(dim):
                esym[i, :, :, i, a] += 0.5 * G[:, :, a].T
                esym[i, :, :, a, i] += 0.5 * G[:, :, a].T
        e2 = np.einsum("inqab,inqab->inq", esym, esym)
        tr = np.einsum("inqaa->inq", esym)
        base = 2.0 * m.mu * e2 + m.lam * tr ** 2
        if self.split == NOSPLIT:
            du = np.einsum("q,cq,inq->cin", sp_.JxW, self.gk_rho, base)
        else:
            du = np.einsum("q,cq,inq->cin", sp_.JxW, self.rho, base)
            du += np.einsum("q,cq,cqabgd,inqab,inqgd->cin", sp_.JxW, self.gkm1_rho,
                            self.tangent, esym, esym)
        dphi = np.einsum("q,cq,qn->cn", sp_.JxW, self.a, sp_.N ** 2)
        dphi = dphi + self.k_phi * np.einsum("q,qnj,qnj->n", sp_.JxW, G, G)[None, :]
        out = sp_.scatter(np.concatenate([du, dphi[:, None, :]], axis=1))
        out[self.constrained] = 1.0
        return out


def residual(tables, state, constrained, material, split=NOSPLIT):
    """Semilinear form A(U), constrained rows zeroed (model.py:420-460)."""
    sp_, m, dim = tables, material, tables.dim
    loc = sp_.gather(state.U)
    gu = sp_.vec_grad_at_qp(loc[:, :dim])
    eu = 0.5 * (gu + np.swapaxes(gu, -1, -2))
    div = np.trace(gu, axis1=-2, axis2=-1)
    phi_q = sp_.at_qp(loc[:, dim])
    gphi = sp_.grad_at_qp(loc[:, dim])
    phit = sp_.at_qp(np.asarray(state.phi_tilde)[sp_.mesh.cells])
    rho = (np.asarray(m.modulus_field(sp_.qp_coords), dtype=float)
           if m.modulus_field is not None else np.ones_like(phi_q))
    p = m.pressure(state.t)
    gk = degradation(phit, m.kappa)
    Ep, _, sp, sm, _ = split_quantities(eu, split, m.lam, m.mu, band=m.split_band)
    stress = ((gk * rho)[..., None, None] * sp + rho[..., None, None] * sm
              + (np.square(phit) * p)[..., None, None] * np.eye(dim))
    out_u = np.einsum("q,cqij,qnj->cin", sp_.JxW, stress, sp_.gradN)
    vphi = ((1.0 - m.kappa) * phi_q * rho * Ep + 2.0 * p * phi_q * div
            - m.g_c / m.eps * (1.0 - phi_q))
    out_phi = np.einsum("q,cq,qn->cn", sp_.JxW, vphi, sp_.N)
    out_phi += m.g_c * m.eps * np.einsum("q,cqj,qnj->cn", sp_.JxW, gphi, sp_.gradN)
    out = sp_.scatter(np.concatenate([out_u, out_phi[:, None, :]], axis=1))
    out[np.asarray(constrained, dtype=bool)] = 0.0
    return out


def crack_energy(tables, U, material):
    """model.py:472-480."""
    loc_phi = tables.gather(U)[:, tables.dim]
    phi_q = tables.at_qp(loc_phi)
    g = tables.grad_at_qp(loc_phi)
    dens = np.square(1.0 - phi_q) / material.eps + material.eps * np.einsum("cqj,cqj->cq", g, g)
    return 0.5 * material.g_c * float(np.einsum("q,cq->", tables.JxW, dens))


def bulk_energy(tables, state, material, split=NOSPLIT):
    """model.py:483-497 (U's own phase field degrades)."""
    dim = tables.dim
    loc = tables.gather(state.U)
    gu = tables.vec_grad_at_qp(loc[:, :dim])
    e = 0.5 * (gu + np.swapaxes(gu, -1, -2))
    div = np.trace(gu, axis1=-2, axis2=-1)
    phi_q = tables.at_qp(loc[:, dim])
    rho = (np.asarray(material.modulus_field(tables.qp_coords), dtype=float)
           if material.modulus_field is not None else np.ones_like(phi_q))
    Ep, Em, _, _, _ = split_quantities(e, split, material.lam, material.mu, band=material.split_band)
    dens = (degradation(phi_q, material.kappa) * rho * Ep + rho * Em
            + np.square(phi_q) * material.pressure(state.t) * div)
    return float(np.einsum("q,cq->", tables.JxW, dens))


def fracture_volume(tables, U):
    """model.py:500-504."""
    phi_q = tables.at_qp(tables.gather(U)[:, tables.dim])
    return float(np.einsum("q,cq->", tables.JxW, 1.0 - phi_q))

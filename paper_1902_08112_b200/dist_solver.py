"""Slab-sharded GMG-preconditioned GMRES across GPUs.

One rank per GPU.  Every level is cut into nested slabs of vertex planes
(`distributed.SlabPartition`); levels too thin to give every rank two cell
layers are replicated and solved redundantly (no communication below the
first sharded level except one all-reduce that agglomerates the restricted
residual).  The per-rank compute is the same libpffmg kernels as on one GPU,
run on the rank's slab lattice (`own_lo/own_hi/plane0` of pffmg_lattice):

* every stencil kernel (block vmults / Chebyshev steps, V-cycle residual,
  restriction, prolongation) is preceded by a ghost-plane halo exchange of
  its input (NCCL send/recv of one plane per neighbour and component);
* inner products sum the owned planes and all-reduce one scalar (GMRES
  MGS, CG-Lanczos), so every rank sees identical Krylov scalars and the
  same iteration count as a single GPU up to rounding;
* the control flow is the reference's (krylov.py:50-136, mgsolve.py:82-283).
"""
from __future__ import annotations

import copy

import numpy as np
import torch

from . import _lib
from .arrays import empty, flags_buffer, host, pack_flags, zeros
from .distributed import (Halo, SlabMesh, SlabPartition, SlabSpace, allreduce_, local_info, owned_slices,
                          to_local)
from .krylov import NoConvergence, SolverControl, lanczos_extremes, probe_vector
from .lattice import device_lattice, info_from_mesh

from .model import DeviceMask, LinearizationState, PhaseFieldOperator


class _Level:
    def __init__(self, l, info_g, slab, rank, world, group):
        self.l = l
        self.slab = slab
        self.info_g = info_g
        self.dim = info_g.dim
        self.nc = info_g.dim + 1
        if slab.replicated or world == 1:
            self.info = copy.copy(info_g)
            self.info.own = (0, 0)
            self.info.plane_lo = 0
        else:
            self.info = local_info(info_g, slab)
        self.mesh = SlabMesh(self.info)
        self.space = SlabSpace(self.mesh, l)
        self.lat = device_lattice(self.mesh)
        self.V = self.info.n_vertices
        self.n = self.nc * self.V
        self.halo = Halo(self.info, slab, rank, world, group)
        self.owned = owned_slices(self.nc, self.info)
        self.sharded = not (slab.replicated or world == 1)


class DistGMG:
    """Distributed level hierarchy + V(1,1) cycle + GMRES for one Newton step."""

    def __init__(self, levels, world, rank, group=None, min_layers=2, degree=4, coarse_target=1e-3,
                 coarse_cap=30, eig_iters=10, seed=0):
        self.world, self.rank, self.group = world, rank, group
        infos = [info_from_mesh(m) for m in levels]
        self.dim = infos[0].dim
        self.part = SlabPartition([int(i.ncell[-1]) for i in infos], world, rank, min_layers,
                                  order=getattr(infos[0], "order", 1))
        self.L = [_Level(l, infos[l], self.part.slab(l), rank, world, group) for l in range(len(levels))]
        self.degree, self.target, self.cap = degree, coarse_target, coarse_cap
        self.eig_iters, self.seed = eig_iters, seed
        # restriction into a replicated level from a sharded one: the coarse
        # lattice restricted to this rank's nested planes (a "virtual slab")
        self.virt = {}
        for l in range(1, len(levels)):
            f, c = self.L[l], self.L[l - 1]
            if f.sharded and not c.sharded:
                vi = copy.copy(c.info_g)
                # coarse plane zc goes to the rank owning fine plane 2 zc, whose
                # stored planes then cover the stencil 2 zc - 1 .. 2 zc + 1
                vi.own = ((f.slab.own_lo + 1) // 2, (f.slab.own_hi + 1) // 2)
                vi.plane_lo = 0
                self.virt[l - 1] = device_lattice(SlabMesh(vi))

    # --------------------------------------------------------------- helpers
    def dot_dev(self, lev, x, y):
        """Owned-dof inner product as a 1-element CUDA tensor, all-reduced (no host sync)."""
        t = torch.zeros(1, dtype=torch.float64, device=x.device)
        for s in lev.owned:
            t += torch.dot(x[s], y[s])
        if lev.sharded:
            allreduce_(t, self.group)
        return t

    def dot(self, lev, x, y):
        t = torch.zeros(1, dtype=torch.float64, device=x.device)
        for s in lev.owned:
            t += torch.dot(x[s], y[s])
        if lev.sharded:
            allreduce_(t, self.group)
        return float(t.item())

    def _inject(self, l, fine_vec, coarse_vec, ncomp, flags=False):
        """Coarse := fine at coincident vertices (owned coarse planes), then ghosts."""
        f, c = self.L[l + 1], self.L[l]
        clat = c.lat if c.sharded or not f.sharded else self.virt[l]
        if flags:
            _lib.call("pffmg_inject_flags", clat.ref, f.lat.ref, _lib.ptr(fine_vec), _lib.ptr(coarse_vec),
                      _lib.stream())
        else:
            _lib.call("pffmg_inject_f64", clat.ref, f.lat.ref, ncomp, _lib.ptr(fine_vec), _lib.ptr(coarse_vec),
                      _lib.stream())
        if c.sharded:
            if flags:
                t = coarse_vec.to(torch.float64)
                c.halo.exchange(t, 1)
                coarse_vec.copy_(t.to(torch.uint8))
            else:
                c.halo.exchange(coarse_vec, ncomp)
        elif f.sharded:                                         # agglomerate onto every rank
            if flags:
                t = coarse_vec.to(torch.float64)
                allreduce_(t, self.group)
                coarse_vec.copy_(t.to(torch.uint8))
            else:
                allreduce_(coarse_vec, self.group)

    # ----------------------------------------------------------------- setup
    def setup(self, state, active, dirichlet, params, split):
        """Level contexts from global finest-level data (mgsolve.py:154-197)."""
        top = self.L[-1]
        nc = top.nc
        g = lambda v, k: torch.as_tensor(to_local(np.asarray(v) if not torch.is_tensor(v) else v, k,
                                                  top.info_g, top.slab), device="cuda")  # noqa: E731
        if not top.sharded:
            g = lambda v, k: torch.as_tensor(np.asarray(v) if not torch.is_tensor(v) else v,  # noqa: E731
                                             device="cuda")
        fine_bool = np.asarray(dirichlet.is_constrained, bool) | np.asarray(active, bool)
        U = [None] * len(self.L)
        PT = [None] * len(self.L)
        FL = [None] * len(self.L)
        U[-1] = g(state.U, nc).to(torch.float64).contiguous()
        PT[-1] = g(state.phi_tilde, 1).to(torch.float64).contiguous()
        FL[-1] = pack_flags(g(fine_bool, nc).to(torch.uint8), nc, top.V)
        for l in range(len(self.L) - 2, -1, -1):
            c = self.L[l]
            U[l], PT[l], FL[l] = zeros(c.n), zeros(c.V), flags_buffer(c.V)
            self._inject(l, U[l + 1], U[l], nc)
            self._inject(l, PT[l + 1], PT[l], 1)
            self._inject(l, FL[l + 1], FL[l], 1, flags=True)
        self.ops, self.inv = [], []
        for l, lev in enumerate(self.L):
            st = LinearizationState(U=U[l], U_prev1=U[l], U_prev2=U[l], t=state.t, t_prev1=state.t_prev1,
                                    t_prev2=state.t_prev2, phi_tilde=PT[l])
            op = PhaseFieldOperator(lev.space, st, DeviceMask(FL[l], nc, lev.V), params, split, _flags=FL[l])
            diag = torch.ones(lev.n, dtype=torch.float64, device="cuda")
            op.diagonal_dev(diag)
            self.ops.append(op)
            self.inv.append(torch.reciprocal(diag))
            lev.flags = FL[l]
            lev.diag = diag
        recs = [self._cg_records(l) for l in range(len(self.L))]
        host_recs = host(torch.stack([t for pair in recs for t in pair]))    # one host sync
        self.spectra = [tuple(self._spectra_from(host_recs[2 * l + k]) for k in range(2))
                        for l in range(len(self.L))]
        self._buffers()
        return self

    def _cg_records(self, l):
        """Jacobi-PCG of both blocks of level l (krylov.py:146-185) with distributed
        dots kept on the device: returns per block the 1 + 2 n scalars
        (rz_0, pAp_1, rz_1, pAp_2, ...) -- no host synchronisation here."""
        lev, op = self.L[l], self.ops[l]
        recs = []
        for k in range(2):
            blk = slice(0, lev.dim * lev.V) if k == 0 else slice(lev.dim * lev.V, lev.n)
            nk = lev.dim if k == 0 else 1
            # the reference's PCG64 probe over the GLOBAL block, sliced to the slab
            ng = nk * lev.info_g.n_vertices
            full = probe_vector(self.seed + 31 * l + 7 * k, ng)
            b = to_local(full, nk, lev.info_g, lev.slab) if lev.sharded else full.clone()
            b = b.contiguous().clone()
            comp0 = 0 if k == 0 else lev.dim
            _lib.call("pffmg_masked_copy", _lib.ptr(lev.flags), lev.V, comp0, nk, _lib.ptr(b), _lib.ptr(b),
                      _lib.stream())
            diag = lev.diag[blk]
            bl = _BlockView(lev, k)
            r = b.clone()
            z = r / diag
            p = z.clone()
            Ap = torch.empty_like(p)
            rz = bl.dot_dev(self, r, z)
            rec = [rz]
            for _ in range(self.eig_iters):
                lev.halo.exchange(p, nk)
                op.apply_dev(k, p, Ap, pre=True)
                pAp = bl.dot_dev(self, p, Ap)
                r = r - (rz / pAp) * Ap
                z = r / diag
                rz_new = bl.dot_dev(self, r, z)
                p = z + (rz_new / rz) * p
                rec += [pAp, rz_new]
                rz = rz_new
            recs.append(torch.cat(rec))
        return recs

    def _spectra_from(self, rec):
        """The reference's breakdown rules replayed on the recorded scalars (krylov.py:168-198)."""
        rz = rec[0]
        al, be = [], []
        for it in range(self.eig_iters):
            if rz <= 0.0 or not np.isfinite(rz):
                break
            pAp = rec[1 + 2 * it]
            if pAp <= 0.0 or not np.isfinite(pAp):
                break
            al.append(rz / pAp)
            rz_new = rec[2 + 2 * it]
            if rz_new <= 1e-28 * rz or not np.isfinite(rz_new):
                break
            be.append(rz_new / rz)
            rz = rz_new
        scal = np.zeros(8 + 128)
        scal[4], scal[5] = len(al), len(be)
        scal[8:8 + len(al)] = al
        scal[8 + 64:8 + 64 + len(be)] = be
        return lanczos_extremes(scal, self.eig_iters)

    def _buffers(self):
        from .mgsolve import LevelContext, _NativeCycle
        ctxs = [LevelContext(l, self.ops[l], lev.diag, self.spectra[l], None, None, lev.flags, inv=self.inv[l])
                for l, lev in enumerate(self.L)]
        # the single-GPU V-cycle (block-diagonal smoothing, device-resident
        # Chebyshev coefficients, one-launch coarse solve) with this object as
        # its communication layer (halo / restrict / prolongate below)
        self.cycle = _NativeCycle(ctxs, self.degree, self.target, self.cap, comm=self)

    # ------------------------------------------------- communication layer
    def halo(self, l, vec, n_comp):
        """Refresh the ghost planes of a level-l vector (no-op on replicated levels)."""
        lev = self.L[l]
        if lev.sharded:
            lev.halo.exchange(vec, n_comp, persistent=True)     # level buffers of the cycle

    def restrict(self, l, fine, coarse, n_comp, comp0):
        """coarse (level l) = masked P^T fine (level l+1); agglomerated into a replicated level."""
        f, c = self.L[l + 1], self.L[l]
        self.halo(l + 1, fine, n_comp)
        clat = c.lat if (c.sharded or not f.sharded) else self.virt[l]
        agglomerate = f.sharded and not c.sharded
        if agglomerate:
            coarse.zero_()
        _lib.call("pffmg_restrict", clat.ref, f.lat.ref, n_comp, comp0, _lib.ptr(fine), _lib.ptr(coarse),
                  _lib.ptr(c.flags), _lib.stream())
        if agglomerate:
            allreduce_(coarse, self.group)

    def prolongate(self, l, coarse, fine, n_comp, comp0):
        """fine (level l+1) += masked P coarse (level l)."""
        f, c = self.L[l + 1], self.L[l]
        self.halo(l, coarse, n_comp)
        _lib.call("pffmg_prolongate", c.lat.ref, f.lat.ref, n_comp, comp0, _lib.ptr(coarse), _lib.ptr(fine),
                  _lib.ptr(f.flags), 1, _lib.stream())

    # --------------------------------------------------------------- V-cycle
    def vcycle(self, r, out):
        """V(1,1) on a local fine residual (mgsolve.py:262-283, FULL); owned rows of `out`."""
        self.cycle.run("full", r, out)
        return out

    def apply(self, v, out):
        top = self.L[-1]
        top.halo.exchange(v, top.nc)
        self.ops[-1].apply_dev(_lib.FULL, v, out)
        return out

    # ----------------------------------------------------------------- GMRES
    def gmres(self, b, control=None):
        """krylov.py:50-136 with distributed inner products; b, x are local slabs."""
        ctl = control or SolverControl()
        top = self.L[-1]
        n = b.numel()
        x = zeros(n)
        r = b.clone()
        rn = float(np.sqrt(self.dot(top, r, r)))
        tol = max(ctl.abs_tol, ctl.rel_tol * rn)
        if rn <= tol:
            return x, 0
        total = 0
        m = int(ctl.restart)
        V = torch.zeros((m + 1, n), dtype=torch.float64, device="cuda")
        Z = torch.zeros((m, n), dtype=torch.float64, device="cuda")
        while True:
            m = min(int(ctl.restart), int(ctl.max_iters) - total)
            if m <= 0:
                raise NoConvergence(x, rn, total)
            H = np.zeros((m + 1, m))
            cs, sn, gg = np.zeros(m), np.zeros(m), np.zeros(m + 1)
            V[0] = r / rn
            gg[0] = rn
            used = 0
            for j in range(m):
                self.vcycle(V[j], Z[j])
                w = V[j + 1]
                self.apply(Z[j], w)
                total += 1
                # MGS (krylov.py:93-107) with the dots kept on the device: each
                # pass all-reduces one scalar and subtracts without a host round
                # trip; the host reads the Hessenberg column once per pass set
                w0 = self.dot_dev(top, w, w)
                hs = []
                for i in range(j + 1):
                    h = self.dot_dev(top, V[i], w)
                    w.sub_(h * V[i])
                    hs.append(h)
                nrm = self.dot_dev(top, w, w)
                vals = host(torch.cat(hs + [w0, nrm]))
                H[:j + 1, j] = vals[:j + 1]
                w0, nrm = float(np.sqrt(vals[-2])), float(np.sqrt(vals[-1]))
                if nrm < 1e-3 * w0:
                    hs = []
                    for i in range(j + 1):
                        cc = self.dot_dev(top, V[i], w)
                        w.sub_(cc * V[i])
                        hs.append(cc)
                    nrm = self.dot_dev(top, w, w)
                    vals = host(torch.cat(hs + [nrm]))
                    H[:j + 1, j] += vals[:j + 1]
                    nrm = float(np.sqrt(vals[-1]))
                H[j + 1, j] = nrm
                brk = H[j + 1, j] == 0.0
                if not brk:
                    w /= H[j + 1, j]
                for i in range(j):
                    t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                    H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                    H[i, j] = t
                den = np.hypot(H[j, j], H[j + 1, j])
                cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
                H[j, j], H[j + 1, j] = den, 0.0
                gg[j + 1] = -sn[j] * gg[j]
                gg[j] = cs[j] * gg[j]
                used = j + 1
                if abs(gg[j + 1]) <= tol or brk:
                    break
            y = np.zeros(used)
            for i in range(used - 1, -1, -1):
                y[i] = (gg[i] - H[i, i + 1:used] @ y[i + 1:]) / H[i, i]
            x += torch.as_tensor(y, device="cuda") @ Z[:used]
            self.apply(x, r)
            r = b - r
            rn = float(np.sqrt(self.dot(top, r, r)))
            if rn <= tol * (1.0 + 1e-8):
                return x, total
            if total >= ctl.max_iters:
                raise NoConvergence(x, rn, total)

    def to_local(self, vec, l=-1):
        lev = self.L[l]
        if not lev.sharded:
            return torch.as_tensor(np.asarray(vec), device="cuda").clone()
        return torch.as_tensor(to_local(np.asarray(vec), lev.nc, lev.info_g, lev.slab), device="cuda")

    def owned_global(self, x_local, l=-1):
        """(global offset, owned values per component) of a local vector."""
        lev = self.L[l]
        return [host(x_local[s]) for s in lev.owned]


class _BlockView:
    """Owned slices of one block (k = 0 displacement, 1 phase field) of a level."""

    def __init__(self, lev, k):
        nk = lev.dim if k == 0 else 1
        offs = lev.info.plane_offsets()
        lo, hi = lev.info.own if lev.info.own != (0, 0) else (0, lev.info.n_planes)
        a, b = int(offs[lo]), int(offs[hi])
        self.slices = [slice(c * lev.V + a, c * lev.V + b) for c in range(nk)]
        self.sharded = lev.sharded

    def dot_dev(self, solver, x, y):
        t = torch.zeros(1, dtype=torch.float64, device=x.device)
        for s in self.slices:
            t += torch.dot(x[s], y[s])
        if self.sharded:
            allreduce_(t, solver.group)
        return t

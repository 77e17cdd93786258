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
* inner products are libpffmg reductions over the rank's OWNED rows
  (pffmg_dot_owned / pffmg_cg_dist / pffmg_multi_dot_owned) followed by one
  all-reduce of the partials: CG-Lanczos takes 2 all-reduces per iteration
  with alpha / beta and the breakdown rules applied on the device
  (pffmg_cg_dist_finish), the Arnoldi step is CGS2 -- two classical
  Gram-Schmidt passes, each one fused multi-dot and one all-reduce of the
  whole column, then the norm -- 3 all-reduces per step instead of the j+2
  sequential ones of distributed MGS (the single-GPU path keeps the
  reference's MGS); every rank sees identical Krylov scalars, and the
  iteration counts equal the single-GPU ones up to rounding;
* the control flow is the reference's (krylov.py:50-136, mgsolve.py:82-283).
"""
from __future__ import annotations

import copy
import os

import numpy as np
import torch

from . import _lib
from .arrays import empty, flags_buffer, host, pack_flags, zeros
from .distributed import (Halo, SlabMesh, SlabPartition, SlabSpace, allreduce_, local_info, owned_slices,
                          to_local)
from .krylov import CG_MAXIT, NoConvergence, SolverControl, lanczos_extremes, probe_vector
from .lattice import device_lattice, info_from_mesh

from .model import DeviceMask, LinearizationState, PhaseFieldOperator


# overlap the ghost-plane exchange of the V-cycle stencils with their interior
# planes (PFFMG_DIST_OVERLAP=0: exchange, then the whole stencil)
OVERLAP = os.environ.get("PFFMG_DIST_OVERLAP", "1") != "0"

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
        # owned vertex range [own_a, own_b) of the rank-local numbering (owned-row reductions)
        offs = self.info.plane_offsets()
        lo, hi = self.info.own if tuple(self.info.own) != (0, 0) else (0, self.info.n_planes)
        self.own_ab = (int(offs[lo]), int(offs[hi]))


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
    def dot_dev(self, lev, x, y, out=None):
        """Owned-row inner product (pffmg_dot_owned), all-reduced; a 1-element
        device tensor (no host sync)."""
        t = out if out is not None else torch.zeros(1, dtype=torch.float64, device=x.device)
        a, b = lev.own_ab
        _lib.call("pffmg_dot_owned", _lib.ptr(x), _lib.ptr(y), x.numel(), lev.V, a, b, _lib.ptr(t),
                  _lib.stream())
        if lev.sharded:
            allreduce_(t, self.group)
        return t

    def dot(self, lev, x, y):
        return float(self.dot_dev(lev, x, y).item())

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
        self.spectra = [tuple(lanczos_extremes(host_recs[2 * l + k], self.eig_iters) for k in range(2))
                        for l in range(len(self.L))]
        self._buffers()
        return self

    def _cg_records(self, l):
        """Jacobi-PCG of both blocks of level l (krylov.py:146-185) on the device:
        owned-row partial sums (pffmg_cg_dist), one all-reduce per reduction
        (2 per iteration), alpha / beta and the breakdown rules applied on the
        device (pffmg_cg_dist_finish).  Returns the two scalar records (the
        layout of pffmg_cg_step) -- no host synchronisation here."""
        lev, op = self.L[l], self.ops[l]
        recs = []
        a, b_ = lev.own_ab
        st = _lib.stream()
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
                      st)
            diag = lev.diag[blk]
            n = b.numel()
            r, z, p, Ap = empty(n), empty(n), empty(n), empty(n)
            scal = torch.zeros(8 + 2 * CG_MAXIT, dtype=torch.float64, device="cuda")

            def phase(ph, src):
                _lib.call("pffmg_cg_dist", ph, _lib.ptr(src), _lib.ptr(diag), _lib.ptr(r), _lib.ptr(z),
                          _lib.ptr(p), n, lev.V, a, b_, _lib.ptr(scal), st)
                if ph < 3:
                    if lev.sharded:
                        slot = (0, 6, 7)[ph]
                        allreduce_(scal[slot:slot + 1], self.group)
                    _lib.call("pffmg_cg_dist_finish", _lib.ptr(scal), ph, st)

            phase(0, b)
            for _ in range(self.eig_iters):
                lev.halo.exchange(p, nk)
                op.apply_dev(k, p, Ap, pre=True)
                phase(1, Ap)
                phase(2, Ap)
                phase(3, Ap)
            recs.append(scal)
        return recs

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

    def overlap_plan(self, l):
        """Row scopes (interior, [boundary...]) of a halo-overlapped stencil on
        level l (PhaseFieldOperator.scope), or None when the level is
        replicated or too thin to have interior planes.  Q1: interior planes
        [lo+1, hi-1) read no ghost plane, the two boundary planes go in one
        PFFMG_HINT_ENDS launch; Q2: node rows [lo+1, hi-2), then [lo, lo+1)
        and [hi-2, hi) (as DistributedOperator.apply_local)."""
        lev = self.L[l]
        if not lev.sharded or not OVERLAP:
            return None
        lo, hi = lev.info.own
        if hi - lo < 4:
            return None
        if getattr(lev.info, "order", 1) == 2:
            return ("rows", lo + 1, hi - 2), [("rows", lo, lo + 1), ("rows", hi - 2, hi)]
        return ("rows", lo + 1, hi - 1), ["ends"]

    def halo_start(self, l, vec, n_comp):
        return self.L[l].halo.start(vec, n_comp, persistent=True)

    def halo_finish(self, l, handle):
        self.L[l].halo.finish(handle)

    def restrict(self, l, fine, coarse, n_comp, comp0):
        """coarse (level l) = masked P^T fine (level l+1); agglomerated into a replicated level."""
        f, c = self.L[l + 1], self.L[l]
        self.halo(l + 1, fine, n_comp)
        clat = c.lat if (c.sharded or not f.sharded) else self.virt[l]
        agglomerate = f.sharded and not c.sharded
        if agglomerate:
            _lib.call("pffmg_scale", 0.0, _lib.ptr(coarse), coarse.numel(), _lib.stream())
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
    def _arnoldi(self, top, V, j, hcol, scr):
        """CGS2 Arnoldi step on w = V[j+1] (krylov.py:93-110 with classical
        Gram-Schmidt twice): pass p: c = V_{0..j} . w over owned rows (fused
        multi-dot), all-reduce the column, w -= V c, H[:, j] += c; then
        ||w|| (fused into the second subtraction), all-reduce, V[j+1] = w / ||w||."""
        a, b = top.own_ab
        n = V.shape[1]
        w = V[j + 1]
        st = _lib.stream()
        for ps in range(2):
            _lib.call("pffmg_multi_dot_owned", _lib.ptr(V), V.stride(0), 0, j + 1, _lib.ptr(w), 0, n, top.V,
                      a, b, _lib.ptr(scr), st)
            if top.sharded:
                allreduce_(scr[:j + 1], self.group)
            _lib.call("pffmg_gs_subtract", _lib.ptr(V), V.stride(0), j + 1, _lib.ptr(scr), _lib.ptr(w), n,
                      _lib.ptr(hcol), top.V, a, b, _lib.ptr(scr[j + 1:]) if ps == 1 else None, st)
        if top.sharded:
            allreduce_(scr[j + 1:j + 2], self.group)
        _lib.call("pffmg_normalize", _lib.ptr(w), _lib.ptr(w), n, _lib.ptr(scr[j + 1:]), _lib.ptr(hcol[j + 1:]), st)

    def gmres(self, b, control=None):
        """krylov.py:50-136 with distributed inner products; b, x are local slabs.
        All vector work is libpffmg kernels (owned-row reductions, CGS2 Arnoldi,
        multi-axpy); the host reads one Hessenberg column per step."""
        ctl = control or SolverControl()
        top = self.L[-1]
        n = b.numel()
        x = zeros(n)
        r = b.clone()
        st = _lib.stream()
        s2 = torch.zeros(1, dtype=torch.float64, device="cuda")
        rn = float(np.sqrt(self.dot_dev(top, r, r, s2).item()))
        tol = max(ctl.abs_tol, ctl.rel_tol * rn)
        if rn <= tol:
            return x, 0
        total = 0
        m = int(ctl.restart)
        V = torch.zeros((m + 1, n), dtype=torch.float64, device="cuda")
        Z = torch.zeros((m, n), dtype=torch.float64, device="cuda")
        Hd = torch.zeros((m, m + 1), dtype=torch.float64, device="cuda")
        scr = torch.zeros(m + 2, dtype=torch.float64, device="cuda")
        yd = torch.zeros(m, dtype=torch.float64, device="cuda")
        while True:
            m = min(int(ctl.restart), int(ctl.max_iters) - total)
            if m <= 0:
                raise NoConvergence(x, rn, total)
            H = np.zeros((m + 1, m))
            cs, sn, gg = np.zeros(m), np.zeros(m), np.zeros(m + 1)
            _lib.call("pffmg_normalize", _lib.ptr(r), _lib.ptr(V[0]), n, _lib.ptr(s2), None, st)   # krylov.py:72
            gg[0] = rn
            _lib.call("pffmg_scale", 0.0, _lib.ptr(Hd), Hd.numel(), st)
            used = 0
            for j in range(m):
                self.vcycle(V[j], Z[j])
                self.apply(Z[j], V[j + 1])
                total += 1
                self._arnoldi(top, V, j, Hd[j], scr)
                H[:j + 2, j] = host(Hd[j, :j + 2])
                brk = H[j + 1, j] == 0.0
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
            yd[:used].copy_(torch.from_numpy(y))
            _lib.call("pffmg_multi_axpy", _lib.ptr(Z), Z.stride(0), used, _lib.ptr(yd), _lib.ptr(x), n, st)
            self.apply(x, r)
            _lib.call("pffmg_sub", _lib.ptr(b), _lib.ptr(r), _lib.ptr(r), n, st)          # r = b - A x
            rn = float(np.sqrt(self.dot_dev(top, r, r, s2).item()))
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

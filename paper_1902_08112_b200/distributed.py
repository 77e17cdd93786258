"""Slab decomposition of a level across ranks.

The lattice is cut along its last axis (y in 2D, z in 3D) into contiguous
slabs of vertex planes.  Rank r *owns* planes [own_lo, own_hi) and stores
planes [own_lo - 1, own_hi] (ghost planes included when they exist), so the
fused operator kernel can compute every cell layer touching an owned plane
and finalise exactly the owned rows (`pffmg_lattice.own_lo/own_hi`).  Before
each stencil application the ghost planes of the input are refreshed by a
halo exchange: each rank sends its first owned plane down and its last owned
plane up -- one plane per neighbour and component, the only data-path
communication of a vmult.  Inner products sum the owned planes locally
(deterministic device reduction) and all-reduce one small vector.

Partitions of a hierarchy are nested: level l+1 owns planes [2a, 2b) when
level l owns [a, b) (the last rank also owns the closing plane), so
injection is rank-local and restriction/prolongation only need the ghost
planes that the halo exchange already provides.  Levels too thin to give
every rank `min_layers` cell layers are replicated on every rank.

Q2 levels (order 2, BASELINE configs[2]) are cut the same way in cell
layers, but their planes are NODE rows (two per cell layer): rank r owns
node rows [2a, 2b) and stores four ghost rows below (the 3x3-node cells of
the layer below need two, the Q2 restriction stencil reaches three) and one
above.

Communication goes through torch.distributed (NCCL over NVLink on GPUs,
gloo on CPUs for the tests); the per-rank compute is a pluggable "local
operator" (the CUDA PhaseFieldOperator on the slab by default).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .lattice import LatticeInfo, info_from_mesh


@dataclass
class Slab:
    """One rank's share of one level."""
    n_cells: int          # cell layers of the level along the cut axis
    own_lo: int           # owned vertex planes [own_lo, own_hi) (global numbers)
    own_hi: int
    lo: int               # stored planes [lo, hi] (owned + ghosts)
    hi: int
    replicated: bool = False
    ghost_lo: int = 1     # ghost planes stored below own_lo (when there is a lower neighbour)

    @property
    def has_lower(self):
        return self.lo < self.own_lo

    @property
    def has_upper(self):
        return self.hi >= self.own_hi


def split_layers(n, world):
    """Balanced cut points c_0 = 0 <= ... <= c_world = n."""
    return [(n * r) // world for r in range(world + 1)]


class SlabPartition:
    """Nested slab partition of a hierarchy with `n_cells[l]` cell layers on level l."""

    def __init__(self, n_cells, world, rank, min_layers=2, order=1):
        self.world, self.rank = world, rank
        self.order = order
        self.n_cells = list(n_cells)
        L = len(self.n_cells)
        # coarsest level that gives every rank at least min_layers layers
        self.first_sharded = L - 1
        for l in range(L):
            if self.n_cells[l] >= min_layers * world:
                self.first_sharded = l
                break
        ls = self.first_sharded
        cuts = split_layers(self.n_cells[ls], world)
        self.slabs = []
        q = 2 if order == 2 else 1                  # planes per cell layer
        gl = 4 if order == 2 else 1
        for l in range(L):
            n = self.n_cells[l]
            N = q * n                                # index of the last plane
            if l < ls or world == 1:
                self.slabs.append(Slab(n, 0, N + 1, 0, N, replicated=world > 1, ghost_lo=gl))
                continue
            k = 2 ** (l - ls)
            a, b = q * cuts[rank] * k, q * cuts[rank + 1] * k
            own_hi = b if rank < world - 1 else N + 1
            self.slabs.append(Slab(n, a, own_hi, max(a - gl, 0), min(own_hi, N), ghost_lo=gl))

    def slab(self, l):
        return self.slabs[l]


def local_info(info: LatticeInfo, slab: Slab) -> LatticeInfo:
    """The rank-local lattice (owned + ghost planes) of a global level."""
    return info.slab(slab.lo, slab.hi, (slab.own_lo, slab.own_hi))


class SlabMesh:
    """Minimal mesh object for a rank-local slab (consumed by device_lattice)."""

    def __init__(self, info: LatticeInfo, global_mesh=None):
        self.lattice_info = info
        self.dim = info.dim
        self.n_vertices = info.n_vertices
        self.cell_size = info.h
        self.global_mesh = global_mesh

    @property
    def cell_volume(self):
        return float(np.prod(self.cell_size))


class SlabSpace:
    def __init__(self, mesh, level):
        self.mesh = mesh
        self.level = level


# ---------------------------------------------------------------- vectors

def to_local(vec, n_comp, info_global: LatticeInfo, slab: Slab):
    """Global component-major vector -> the rank's slab (owned + ghosts)."""
    offs = info_global.plane_offsets()
    V = info_global.n_vertices
    a, b = int(offs[slab.lo]), int(offs[slab.hi + 1])
    if isinstance(vec, torch.Tensor):
        return torch.cat([vec[c * V + a:c * V + b] for c in range(n_comp)])
    vec = np.asarray(vec)
    return np.concatenate([vec[c * V + a:c * V + b] for c in range(n_comp)])


def owned_slices(n_comp, info_local: LatticeInfo):
    """Slices of a local vector covering the owned planes, one per component."""
    offs = info_local.plane_offsets()
    V = info_local.n_vertices
    lo, hi = info_local.own
    if lo == 0 and hi == 0:
        lo, hi = 0, info_local.n_planes
    a, b = int(offs[lo]), int(offs[hi])
    return [slice(c * V + a, c * V + b) for c in range(n_comp)]


class Halo:
    """Ghost-plane exchange of component-major local vectors."""

    def __init__(self, info_local: LatticeInfo, slab: Slab, rank, world, group=None):
        self.offs = info_local.plane_offsets()
        self.V = info_local.n_vertices
        self.slab = slab
        self.rank, self.world, self.group = rank, world, group
        lo_own = slab.own_lo - slab.lo          # local index of the first owned plane
        hi_own = slab.own_hi - slab.lo          # one past the last owned plane
        g = slab.ghost_lo                       # the upper neighbour stores g planes of ours
        o = self.offs
        self.send_down = (int(o[lo_own]), int(o[lo_own + 1])) if slab.has_lower else None
        self.recv_down = (int(o[0]), int(o[lo_own])) if slab.has_lower else None
        self.send_up = (int(o[hi_own - g]), int(o[hi_own])) if slab.has_upper else None
        self.recv_up = (int(o[hi_own]), int(o[hi_own + 1])) if slab.has_upper else None
        self._ops = {}

    def exchange(self, vec, n_comp, persistent=False):
        """Refresh ghost planes of `vec` (a 1-D tensor of n_comp * V entries) in place.

        With NCCL the planes go device to device; with gloo (CPU tests, or
        ranks sharing one GPU in tests) CUDA planes are staged through host memory."""
        self.finish(self.start(vec, n_comp, persistent))
        return vec

    def start(self, vec, n_comp, persistent=False):
        """Post the exchange; returns a handle for finish().  Under NCCL the
        transfers run on NCCL's stream, concurrently with work enqueued on the
        current stream afterwards (which must not touch the ghost planes).

        CUDA vectors go as ONE contiguous message per neighbour: the sent
        planes of every component are packed by a libpffmg kernel
        (pffmg_pack_rows) into a persistent buffer, received into another and
        unpacked after the wait (`persistent` is accepted for the callers'
        convenience; the packed path is always persistent).  CPU vectors (the
        oracle-backed CPU tests) go per component."""
        if self.world == 1 or self.slab.replicated:
            return None
        if vec.is_cuda:
            return self._start_packed(vec, n_comp)
        ops = self._build_ops(vec, n_comp, lambda t: t, [])
        return (dist.batch_isend_irecv(ops) if ops else []), []

    def _build_ops(self, vec, n_comp, buf, back):
        ops = []
        V = self.V
        for c in range(n_comp):
            base = c * V
            for send, recv, peer in ((self.send_down, self.recv_down, self.rank - 1),
                                     (self.send_up, self.recv_up, self.rank + 1)):
                if send is None:
                    continue
                a, b = send
                ops.append(dist.P2POp(dist.isend, buf(vec[base + a:base + b]), peer, self.group))
                a, b = recv
                r = buf(vec[base + a:base + b])
                ops.append(dist.P2POp(dist.irecv, r, peer, self.group))
                if r.data_ptr() != vec[base + a:base + b].data_ptr():
                    back.append((vec[base + a:base + b], r))
        return ops

    def _bufs(self, n_comp, device):
        key = (n_comp, str(device))
        b = self._ops.get(key)
        if b is None:
            b = {}
            for name, rng in (("sd", self.send_down), ("rd", self.recv_down), ("su", self.send_up),
                              ("ru", self.recv_up)):
                if rng is not None:
                    b[name] = torch.empty(n_comp * (rng[1] - rng[0]), dtype=torch.float64, device=device)
            self._ops[key] = b
        return b

    def _start_packed(self, vec, n_comp):
        from . import _lib
        stage = _backend(self.group) != "nccl"
        b = self._bufs(n_comp, vec.device)
        s = _lib.stream()
        ops, back = [], []
        for snd, rcv, sk, rk, peer in ((self.send_down, self.recv_down, "sd", "rd", self.rank - 1),
                                       (self.send_up, self.recv_up, "su", "ru", self.rank + 1)):
            if snd is None:
                continue
            _lib.call("pffmg_pack_rows", _lib.ptr(vec), self.V, n_comp, snd[0], snd[1] - snd[0], _lib.ptr(b[sk]),
                      0, s)
            sbuf = b[sk].cpu() if stage else b[sk]
            rbuf = torch.empty(b[rk].numel(), dtype=torch.float64) if stage else b[rk]
            ops.append(dist.P2POp(dist.isend, sbuf, peer, self.group))
            ops.append(dist.P2POp(dist.irecv, rbuf, peer, self.group))
            back.append((rcv, b[rk], rbuf if stage else None))
        reqs = dist.batch_isend_irecv(ops) if ops else []
        return reqs, [("unpack", vec, n_comp, back)]

    def finish(self, handle):
        if handle is None:
            return
        reqs, back = handle
        for req in reqs:
            req.wait()
        for item in back:
            if item[0] == "unpack":
                from . import _lib
                _, vec, n_comp, recvs = item
                for rng, dbuf, hbuf in recvs:
                    if hbuf is not None:                  # gloo: staged through the host
                        dbuf.copy_(hbuf)
                    _lib.call("pffmg_pack_rows", _lib.ptr(vec), self.V, n_comp, rng[0], rng[1] - rng[0],
                              _lib.ptr(dbuf), 1, _lib.stream())
            else:
                dst, src = item
                dst.copy_(src)


def _backend(group=None):
    try:
        return dist.get_backend(group)
    except Exception:
        return "none"


def allreduce_(t, group=None, op=None):
    """In-place sum (or `op`) all-reduce; CUDA tensors staged through the host under gloo."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return t
    op = op or dist.ReduceOp.SUM
    if t.is_cuda and _backend(group) != "nccl":
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)
    return t


def dist_dot(x, y, n_comp, info_local, group=None, local_dot=None):
    """Sum over owned dofs of x*y across ranks (deterministic for a fixed world size)."""
    parts = []
    for s in owned_slices(n_comp, info_local):
        if local_dot is not None:
            parts.append(local_dot(x[s], y[s]))
        else:
            parts.append(torch.dot(x[s], y[s]))
    t = torch.stack([torch.as_tensor(p, dtype=torch.float64, device=x.device) for p in parts]).sum()
    t = t.reshape(1)
    allreduce_(t, group)
    return float(t.item())


class DistributedOperator:
    """Slab-sharded fused vmult of one level.

    `local_factory(space, state, mask, params, split)` builds the per-rank
    compute (default: the CUDA PhaseFieldOperator).  State vectors, masks and
    flags are sliced to the slab once; `apply_local` refreshes the input's
    ghost planes and applies the operator to the owned rows."""

    def __init__(self, global_mesh, level, partition: SlabPartition, state, mask, params, split,
                 local_factory=None, group=None):
        info = info_from_mesh(global_mesh)
        self.info_global = info
        self.slab = partition.slab(level)
        self.info = local_info(info, self.slab)
        self.n_comp = info.dim + 1
        self.rank, self.world = partition.rank, partition.world
        self.halo = Halo(self.info, self.slab, self.rank, self.world, group)
        self.group = group
        nc = self.n_comp
        loc = lambda v, k: to_local(v, k, info, self.slab)  # noqa: E731
        from .model import ConstraintMask, LinearizationState
        st = LinearizationState(U=loc(state.U, nc), U_prev1=loc(state.U_prev1, nc),
                                U_prev2=loc(state.U_prev2, nc), t=state.t, t_prev1=state.t_prev1,
                                t_prev2=state.t_prev2, phi_tilde=loc(state.phi_tilde, 1))
        m = ConstraintMask(loc(mask.is_constrained, nc), loc(mask.inhomogeneity, nc))
        space = SlabSpace(SlabMesh(self.info, global_mesh), level)
        if local_factory is None:
            from .model import PhaseFieldOperator
            local_factory = PhaseFieldOperator
        self.local = local_factory(space, st, m, params, split)
        self.owned = owned_slices(nc, self.info)

    @property
    def n_local(self):
        return self.n_comp * self.info.n_vertices

    def to_local(self, vec):
        return to_local(vec, self.n_comp, self.info_global, self.slab)

    def apply_local(self, v_loc, out_loc):
        """out (owned rows) = G~ v, after refreshing v's ghost planes.

        The halo exchange overlaps the interior rows (their cells read owned
        planes only; NCCL runs on its own stream, gloo stages through the host);
        the two boundary rows run after it lands."""
        lo, hi = self.info.own if self.info.own != (0, 0) else (0, self.info.n_planes)
        if (hasattr(self.local, "apply_rows_dev") and v_loc.is_cuda and self.world > 1
                and hi - lo >= 4 and not self.slab.replicated):
            from . import _lib
            h = self.halo.start(v_loc, self.n_comp, persistent=True)
            if self.info.order == 2:
                # Q2: node row lo+1 is interior to the first owned cell layer; rows
                # hi-2 and hi-1 belong to the top layer, whose cells read ghost row hi
                self.local.apply_rows_dev(_lib.FULL, v_loc, out_loc, lo + 1, hi - 2)
                self.halo.finish(h)
                self.local.apply_rows_dev(_lib.FULL, v_loc, out_loc, lo, lo + 1)
                self.local.apply_rows_dev(_lib.FULL, v_loc, out_loc, hi - 2, hi)
                return out_loc
            self.local.apply_rows_dev(_lib.FULL, v_loc, out_loc, lo + 1, hi - 1)
            self.halo.finish(h)
            self.local.apply_ends_dev(_lib.FULL, v_loc, out_loc)      # rows lo and hi-1, one launch
            return out_loc
        self.halo.exchange(v_loc, self.n_comp)
        if hasattr(self.local, "apply_dev") and v_loc.is_cuda:
            from . import _lib
            self.local.apply_dev(_lib.FULL, v_loc, out_loc)
        else:
            out_loc.copy_(torch.as_tensor(self.local.apply(v_loc), dtype=out_loc.dtype))
        return out_loc

    def dot(self, x, y):
        return dist_dot(x, y, self.n_comp, self.info, self.group)

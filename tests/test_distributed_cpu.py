"""Slab decomposition host logic on CPU with the gloo backend (world size 2
and 3): nested partitions, halo exchange, owned-row vmult equal to the
single-rank operator, distributed inner products.  The per-rank compute is
the CPU oracle injected as the local operator (test infrastructure); on GPUs
the same code drives the CUDA kernel."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.golden.specs import MESHES


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleSlabOperator:
    """Local operator of one slab computed by the CPU oracle."""

    def __init__(self, space, state, mask, params, split):
        from oracle import fe, jacobian
        from oracle.meshgen import OracleLevel, corner_bits
        info = space.mesh.lattice_info
        dim = info.dim
        ext = info.ncell + 1
        # vertices of the slab in local id order (x fastest, rows contiguous)
        if info.rows is None:
            grids = np.meshgrid(*[np.arange(e) for e in ext[::-1]], indexing="ij")
            rel = np.stack([g.ravel() for g in grids[::-1]], axis=1)
            present = np.ones(int(np.prod(ext)), bool)
        else:
            voff, vlo, vhi = info.rows[:3]
            pts = []
            for r in range(len(vlo)):
                y = r % ext[1]
                z = r // ext[1]
                for x in range(vlo[r], vhi[r]):
                    pts.append((x, y, z)[:dim] if dim == 3 else (x, r))
            rel = np.array(pts, dtype=np.int64)
        ids = {tuple(p): i for i, p in enumerate(map(tuple, rel))}
        cells = []
        bits = corner_bits(dim)
        for idx in np.ndindex(*tuple(info.ncell[::-1])):
            c = np.array(idx[::-1])
            corner = [ids.get(tuple(c + b)) for b in bits]
            if all(k is not None for k in corner):
                if info.rows is not None:
                    s = c[1] + (info.ncell[1] * c[2] if dim == 3 else 0)
                    if not (info.rows[3][s] <= c[0] < info.rows[4][s]):
                        continue
                cells.append(corner)
        keys = rel.copy()
        keys[:, -1] += info.plane_lo
        lev = OracleLevel(vertices=keys * info.h, cells=np.array(cells, dtype=np.int64),
                          cell_size=info.h, keys=keys, key_mod=10 ** 6)
        T = fe.LevelTables(lev, space.level)
        mat = jacobian.Material(mu=params.mu, lam=params.lam, g_c=params.g_c, kappa=params.kappa,
                                eps=params.eps, pressure_fn=params.pressure_fn)
        st = jacobian.State(U=np.asarray(state.U), U_prev1=np.asarray(state.U), U_prev2=np.asarray(state.U),
                            t=state.t, t_prev1=0.0, t_prev2=0.0, phi_tilde=np.asarray(state.phi_tilde))
        self.op = jacobian.JacobianOperator(T, st, np.asarray(mask.is_constrained), mat)

    def apply(self, v):
        return self.op.apply(np.asarray(v))


def _problem(name):
    from paper_1902_08112_b200 import lattice
    from paper_1902_08112_b200.model import ConstraintMask, LinearizationState, MaterialParams
    blocks, n_levels, dim = MESHES[name]
    levels = lattice.build_hierarchy(blocks, n_levels, dim)
    fine = levels[-1]
    V = fine.n_vertices
    n = (dim + 1) * V
    rng = np.random.default_rng(5)
    U = 1e-2 * rng.standard_normal(n)
    U[dim * V:] = np.clip(0.6 + 0.4 * rng.standard_normal(V), 0, 1)
    st = LinearizationState(U=U, U_prev1=U, U_prev2=U, t=0.2, t_prev1=0.0, t_prev2=0.0,
                            phi_tilde=U[dim * V:].copy())
    flags = rng.random(n) < 0.1
    mask = ConstraintMask(flags, np.zeros(n))
    params = MaterialParams(mu=1.3, lam=0.9, g_c=0.7, kappa=1e-10, eps=0.5,
                            pressure_fn=lambda t: 10.0 * t)
    v = rng.standard_normal(n)
    return levels, st, mask, params, v


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1902_08112_b200 import distributed as D
        from paper_1902_08112_b200.lattice import info_from_mesh
        from paper_1902_08112_b200.model import SplitKind
        levels, st, mask, params, v = _problem(name)
        n_cells = [int(info_from_mesh(m).ncell[-1]) for m in levels]
        part = D.SlabPartition(n_cells, world, rank, min_layers=2)
        L = len(levels) - 1
        op = D.DistributedOperator(levels[L], L, part, st, mask, params, SplitKind.NOSPLIT,
                                   local_factory=OracleSlabOperator)
        # halo exchange: ghosts of a garbage-initialised local vector get the true values
        v_loc = torch.as_tensor(op.to_local(v))
        true_loc = v_loc.clone()
        for s in D.owned_slices(op.n_comp, op.info):
            pass
        ghost = torch.ones(op.n_local, dtype=torch.bool)
        for s in op.owned:
            ghost[s] = False
        v_loc[ghost] = -7.0
        op.halo.exchange(v_loc, op.n_comp)
        halo_ok = bool(torch.equal(v_loc, true_loc))
        out = torch.zeros(op.n_local, dtype=torch.float64)
        op.apply_local(v_loc, out)
        owned = torch.cat([out[s] for s in op.owned]).numpy()
        d = op.dot(v_loc, v_loc)
        q.put((rank, halo_ok, owned, d, [(s.own_lo, s.own_hi, s.lo, s.hi, s.replicated) for s in part.slabs]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("cfg1", 2), ("cfg1", 3), ("cube", 2), ("lprism", 2),
                                        ("rect3d", 3)])
def test_slab_vmult_matches_single_rank(name, world):
    from oracle import fe, jacobian, meshgen
    from tests.helpers import oracle_levels
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # reference: single-rank oracle on the global mesh
    levels, st, mask, params, v = _problem(name)
    olev = oracle_levels(name)[-1]
    T = fe.LevelTables(olev, len(levels) - 1)
    mat = jacobian.Material(mu=params.mu, lam=params.lam, g_c=params.g_c, kappa=params.kappa,
                            eps=params.eps, pressure_fn=params.pressure_fn)
    ost = jacobian.State(U=st.U, U_prev1=st.U, U_prev2=st.U, t=st.t, t_prev1=0.0, t_prev2=0.0,
                         phi_tilde=st.phi_tilde)
    ref = jacobian.JacobianOperator(T, ost, mask.is_constrained, mat).apply(v)
    dim = olev.dim
    nc = dim + 1
    V = olev.n_vertices
    from paper_1902_08112_b200.lattice import info_from_mesh
    info = info_from_mesh(levels[-1])
    offs = info.plane_offsets()
    got = np.zeros_like(ref)
    covered = np.zeros(ref.size, bool)
    for rank, halo_ok, owned, d, slabs in res:
        assert halo_ok, f"rank {rank} halo"
        own_lo, own_hi = slabs[-1][0], slabs[-1][1]
        a, b = int(offs[own_lo]), int(offs[own_hi])
        per = b - a
        for c in range(nc):
            got[c * V + a:c * V + b] = owned[c * per:(c + 1) * per]
            covered[c * V + a:c * V + b] = True
        assert abs(d - float(v @ v)) <= 1e-12 * float(v @ v)
    assert covered.all()                                    # owned ranges tile the level
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)


def test_partition_is_nested_and_covers():
    from paper_1902_08112_b200.distributed import SlabPartition
    n_cells = [3 * 2 ** l for l in range(8)]                # cfg5: 3 .. 384 layers
    for world in (1, 2, 4, 8):
        parts = [SlabPartition(n_cells, world, r, min_layers=2) for r in range(world)]
        for l, n in enumerate(n_cells):
            owned = np.zeros(n + 1, int)
            for p in parts:
                s = p.slab(l)
                owned[s.own_lo:s.own_hi] += 1
                assert s.lo == max(s.own_lo - 1, 0) and s.hi == min(s.own_hi, n)
            if parts[0].slab(l).replicated:
                assert np.all(owned == world)
            else:
                assert np.all(owned == 1)
                if l > parts[0].first_sharded:
                    for p in parts:                           # nesting
                        c, f = p.slab(l - 1), p.slab(l)
                        assert f.own_lo == 2 * c.own_lo
                        assert f.own_hi == (2 * c.own_hi if c.own_hi <= n_cells[l - 1] else n + 1)


# ------------------------------------------------------------------ Q2 slabs

class OracleQ2SlabOperator:
    """Local operator of one Q2 slab (node rows [lo, hi] of the level) by the
    Q2 CPU oracle: the slab is itself a box of whole cell layers."""

    def __init__(self, space, state, mask, params, split):
        from oracle import jacobian, q2
        info = space.mesh.lattice_info
        g = space.mesh.global_mesh
        h = np.asarray(info.h, float)
        lo = np.asarray(g.lo, float) + np.array([0.0, 0.5 * info.plane_lo * h[1]])
        lev = q2.Q2Level(np.array([int(info.ncell[0]), int(info.ncell[1])]), h, lo)
        T = q2.Q2Tables(lev)
        mat = jacobian.Material(mu=params.mu, lam=params.lam, g_c=params.g_c, kappa=params.kappa,
                                eps=params.eps, pressure_fn=params.pressure_fn)
        st = jacobian.State(U=np.asarray(state.U), U_prev1=np.asarray(state.U), U_prev2=np.asarray(state.U),
                            t=state.t, t_prev1=0.0, t_prev2=0.0, phi_tilde=np.asarray(state.phi_tilde))
        self.op = jacobian.JacobianOperator(T, st, np.asarray(mask.is_constrained), mat)

    def apply(self, v):
        return self.op.apply(np.asarray(v))


def _q2_problem(n_coarse=2, n_levels=3):
    from paper_1902_08112_b200 import lattice
    from paper_1902_08112_b200.model import ConstraintMask, LinearizationState, MaterialParams
    levels = lattice.build_q2_hierarchy(-1.0, 1.0, n_coarse, n_levels)
    V = levels[-1].n_vertices
    n = 3 * V
    rng = np.random.default_rng(8)
    U = 1e-2 * rng.standard_normal(n)
    U[2 * V:] = np.clip(0.6 + 0.4 * rng.standard_normal(V), 0, 1)
    st = LinearizationState(U=U, U_prev1=U, U_prev2=U, t=0.2, t_prev1=0.0, t_prev2=0.0,
                            phi_tilde=U[2 * V:].copy())
    mask = ConstraintMask(rng.random(n) < 0.1, np.zeros(n))
    params = MaterialParams(mu=1.3, lam=0.9, g_c=0.7, kappa=1e-10, eps=0.5, pressure_fn=lambda t: 10.0 * t)
    return levels, st, mask, params, rng.standard_normal(n)


def _q2_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1902_08112_b200 import distributed as D
        from paper_1902_08112_b200.model import SplitKind
        levels, st, mask, params, v = _q2_problem()
        part = D.SlabPartition([int(m.ncell[1]) for m in levels], world, rank, min_layers=2, order=2)
        L = len(levels) - 1
        op = D.DistributedOperator(levels[L], L, part, st, mask, params, SplitKind.NOSPLIT,
                                   local_factory=OracleQ2SlabOperator)
        v_loc = torch.as_tensor(op.to_local(v))
        true_loc = v_loc.clone()
        ghost = torch.ones(op.n_local, dtype=torch.bool)
        for s in op.owned:
            ghost[s] = False
        v_loc[ghost] = -7.0
        op.halo.exchange(v_loc, op.n_comp)
        halo_ok = bool(torch.equal(v_loc, true_loc))
        out = torch.zeros(op.n_local, dtype=torch.float64)
        op.apply_local(v_loc, out)
        owned = torch.cat([out[s] for s in op.owned]).numpy()
        s = part.slab(L)
        q.put((rank, halo_ok, owned, op.dot(v_loc, v_loc), s.own_lo, s.own_hi))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_q2_slab_vmult_matches_single_rank(world):
    """Q2 node-row slabs: 4 ghost rows below / 1 above, halo exchange restores
    them, and the owned rows of every rank stitch to the whole-box Q2 oracle."""
    from oracle import jacobian, q2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_q2_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    levels, st, mask, params, v = _q2_problem()
    g = levels[-1]
    T = q2.Q2Tables(q2.Q2Level(np.asarray(g.ncell), np.asarray(g.cell_size), np.asarray(g.lo)))
    mat = jacobian.Material(mu=params.mu, lam=params.lam, g_c=params.g_c, kappa=params.kappa,
                            eps=params.eps, pressure_fn=params.pressure_fn)
    ost = jacobian.State(U=st.U, U_prev1=st.U, U_prev2=st.U, t=st.t, t_prev1=0.0, t_prev2=0.0,
                         phi_tilde=st.phi_tilde)
    ref = jacobian.JacobianOperator(T, ost, mask.is_constrained, mat).apply(v)
    V = g.n_vertices
    nxn = 2 * int(g.ncell[0]) + 1
    got = np.full(ref.size, np.nan)
    for rank, halo_ok, owned, d, lo, hi in res:
        assert halo_ok, f"rank {rank} halo"
        assert lo % 2 == 0
        a, b = lo * nxn, hi * nxn
        per = b - a
        for c in range(3):
            got[c * V + a:c * V + b] = owned[c * per:(c + 1) * per]
        assert abs(d - float(v @ v)) <= 1e-12 * float(v @ v)
    assert not np.isnan(got).any()
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)


def test_q2_partition_node_rows():
    """Q2 partitions: owned node rows tile 0..2n, start on cell boundaries, nest
    across levels, store 4 ghost rows below and 1 above; the halo ranges pair up."""
    from paper_1902_08112_b200.distributed import Halo, SlabPartition, local_info
    from paper_1902_08112_b200.lattice import build_q2_hierarchy, info_from_mesh
    levels = build_q2_hierarchy(0.0, 1.0, 8, 4)
    n_cells = [int(m.ncell[1]) for m in levels]
    for world in (2, 3, 4):
        parts = [SlabPartition(n_cells, world, r, min_layers=2, order=2) for r in range(world)]
        for l, n in enumerate(n_cells):
            owned = np.zeros(2 * n + 1, int)
            for p in parts:
                s = p.slab(l)
                owned[s.own_lo:s.own_hi] += 1
                assert s.own_lo % 2 == 0 and s.lo % 2 == 0 and s.hi % 2 == 0
                if not s.replicated:
                    assert s.lo == max(s.own_lo - 4, 0) and s.hi == min(s.own_hi, 2 * n)
            assert np.all(owned == (world if parts[0].slab(l).replicated else 1))
            if parts[0].slab(l).replicated:
                continue
            info = info_from_mesh(levels[l])
            nxn = 2 * int(levels[l].ncell[0]) + 1
            halos = []
            for r, p in enumerate(parts):
                s = p.slab(l)
                li = local_info(info, s)
                assert li.n_planes == s.hi - s.lo + 1 and li.n_vertices == li.n_planes * nxn
                halos.append((s, Halo(li, s, r, world)))
            for r in range(world - 1):                   # what r sends up, r+1 receives below
                (s0, h0), (s1, h1) = halos[r], halos[r + 1]
                assert h0.send_up[1] - h0.send_up[0] == h1.recv_down[1] - h1.recv_down[0] == 4 * nxn
                assert h0.send_up[0] // nxn + s0.lo == s1.lo
                assert h1.send_down[1] - h1.send_down[0] == h0.recv_up[1] - h0.recv_up[0] == nxn
                assert h0.recv_up[0] // nxn + s0.lo == s1.own_lo

"""Sharding host logic on CPU: halo plans from the link tables, and the halo
exchange protocol over torch.distributed (gloo, world_size 2) reproducing the
unsharded right-hand side bit for bit with the C oracle."""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1012_4382_b200.shard import TILE, build_shards, shard_bounds, stage_output_buffer, t_end_steps


def _tables(modes, n_max):
    ind, tiers, plus, minus = orc.enumerate_hierarchy(modes, n_max)
    return ind, tiers, plus, minus


def test_shard_bounds_cover_and_balance():
    b = shard_bounds(319770, 8)
    assert b[0] == 0 and b[-1] == 319770
    assert np.max(np.diff(b)) - np.min(np.diff(b)) <= 1
    with pytest.raises(ValueError):
        shard_bounds(3, 4)


@pytest.mark.parametrize("modes,kp1,n_max,shards", [(14, 2, 3, 2), (14, 2, 4, 5), (7, 1, 6, 3),
                                                    (14, 2, 5, 8)])
def test_shard_layouts_are_consistent(modes, kp1, n_max, shards):
    ind, tiers, plus, minus = _tables(modes, n_max)
    n_tot = len(ind)
    L = build_shards(ind, tiers, plus, minus, shards, kp1, n_max)
    owned = np.concatenate([x.local2ref[: x.own_tiles * TILE] for x in L])
    owned = owned[owned >= 0]
    assert np.array_equal(np.sort(owned), np.arange(n_tot))          # a partition
    assert sum(x.root for x in L) == 1 and L[0].root and L[0].local2ref[0] == 0
    for x in L:
        own_slots = x.own_tiles * TILE
        assert x.n_local % TILE == 0 and x.n_local >= own_slots
        slots = np.nonzero(x.local2ref[:own_slots] >= 0)[0]
        ref = x.local2ref[slots]
        # local links name the same ADOs as the reference links
        for loc, glob, none in ((x.plus, plus, -1), (x.minus, minus, -2)):
            lt, gt = loc[slots], glob[ref]
            assert np.all((gt < 0) == (lt < 0)) and np.all(lt[gt < 0] == none)
            assert np.array_equal(x.local2ref[lt[gt >= 0]], gt[gt >= 0])
        assert np.array_equal(x.nvec[slots], ind[ref])
        # whole top-tier tiles past top_tile, nothing of the top tier before it
        top_ref = x.local2ref[x.top_tile * TILE:own_slots]
        assert np.all(tiers[top_ref[top_ref >= 0]] == n_max)
        assert np.all(tiers[x.local2ref[: x.top_tile * TILE][x.local2ref[: x.top_tile * TILE] >= 0]] < n_max)
        # halo: exactly the (neighbour, site) pairs the owned ADOs reach elsewhere
        need = set()
        for m in range(modes):
            for tab in (x.plus, x.minus):
                t = tab[slots, m]
                for v in t[t >= own_slots]:
                    need.add((int(v), m // kp1))
        got = set()
        for o, pos, site in x.recv:
            assert o != x.rank
            assert np.all(pos >= own_slots)
            got |= set(zip(pos.tolist(), site.tolist()))
        assert got == need
        # the owner ships the same (ADO, site) entries in the same order
        for o, pos, site in x.recv:
            (c, spos, ssite), = [e for e in L[o].send if e[0] == x.rank]
            assert np.array_equal(L[o].local2ref[spos], x.local2ref[pos])
            assert np.array_equal(ssite, site) and np.all(spos < L[o].own_tiles * TILE)
        # launch groups partition the owned tiles; halo readers are in groups 2, 3
        g = np.concatenate(x.groups)
        assert np.array_equal(np.sort(g), np.arange(x.own_tiles))
        links = np.concatenate([x.plus[:own_slots], x.minus[:own_slots]], axis=1)
        reads = np.any(links >= own_slots, axis=1).reshape(-1, TILE).any(axis=1)
        assert np.all(reads[np.concatenate([x.groups[2], x.groups[3]])])
        assert not np.any(reads[np.concatenate([x.groups[0], x.groups[1]])])
        sends = np.zeros(x.own_tiles, bool)
        for _, pos, _ in x.send:
            sends[pos // TILE] = True
        assert np.all(sends[np.concatenate([x.groups[0], x.groups[2]])])
        assert not np.any(sends[np.concatenate([x.groups[1], x.groups[3]])])


def test_halo_volume_config4():
    """Config 4 (M = 14, N_max = 8) at P = 8: compressed crosses per stage per
    shard and memory of owned + halo slots only."""
    ind, tiers, plus, minus = _tables(14, 8)
    L = build_shards(ind, tiers, plus, minus, 8, 2, 8)
    assert max(x.halo_bytes_per_stage() for x in L) < 9e6
    assert max(x.n_local for x in L) < 0.4 * len(ind)      # not the full hierarchy
    assert all(x.top_tile < x.own_tiles for x in L)         # paired-round tiles on every shard


def test_stage_buffers_and_steps():
    assert [stage_output_buffer(s) for s in (1, 2, 3, 4)] == [1, 2, 3, 0]
    assert t_end_steps(1000.0, 1.0) == 1000 and t_end_steps(30.0, 1.0) == 30
    assert t_end_steps(0.0, 2.5) == 0 and t_end_steps(10.0, 3.0) == 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cross_worker(rank, world, port, out_q):
    """One shard per process: its owned ADOs, NaN everywhere else; the crosses
    its plan receives come from the owners over gloo (the transport of
    hb_shard_steps); the oracle RHS on the LOCAL tables must equal the global
    RHS on every owned ADO, bit for bit."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1012_4382_b200 as xf
    fmo = xf.build_fmo_system()
    bath = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
    rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
    pb = orc.Problem(fmo, bath, rates, 3, 1)
    L = build_shards(pb.indices, pb.tiers, pb.plus, pb.minus, world, 2, 3)[rank]
    rng = np.random.default_rng(12)
    full = rng.standard_normal((pb.n_tot, 7, 7)) + 1j * rng.standard_normal((pb.n_tot, 7, 7))
    full = full + full.conj().transpose(0, 2, 1)          # Hermitian, like every ADO
    own_slots = L.own_tiles * TILE
    local = np.full((L.n_local, 7, 7), np.nan + 0j)
    ok_own = L.local2ref[:own_slots] >= 0
    local[:own_slots][ok_own] = full[L.local2ref[:own_slots][ok_own]]

    def cross(m, s):  # row and column s of each matrix: the 2d-1 shipped elements
        return np.concatenate([m[s, :], m[:, s]])

    reqs = []
    for dst, pos, site in L.send:
        payload = np.stack([cross(local[p], s) for p, s in zip(pos, site)])
        reqs.append(dist.isend(torch.from_numpy(payload.view(np.float64).copy()), dst))
    for owner, pos, site in L.recv:
        t = torch.empty((len(pos), 28), dtype=torch.float64)
        dist.recv(t, owner)
        got = t.numpy().view(np.complex128)
        for i, (p, s) in enumerate(zip(pos, site)):
            local[p, s, :] = got[i, :7]
            local[p, :, s] = got[i, 7:]
    for r in reqs:
        r.wait()
    rhs_local = orc.rhs_from_arrays(local, pb.h, pb.site_of, L.plus, L.minus, L.nvec.astype(np.int32),
                                    pb.n_sites, pb.kp1, pb.nu, pb.a, pb.b, pb.decay)
    rhs_full = pb.rhs(full)
    slots = np.nonzero(ok_own)[0]
    ok = np.array_equal(rhs_local[slots], rhs_full[L.local2ref[slots]])
    out_q.put((rank, ok, len(slots), L.halo_entries()))
    dist.destroy_process_group()


def test_gloo_cross_halo_exchange_reproduces_unsharded_rhs():
    """only the crosses are shipped; the rest of every halo slot is NaN here, so
    a kernel reading any other element of a neighbour would fail"""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cross_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in res] == [True, True]
    assert sum(r[2] for r in res) == orc.hierarchy_size(14, 3)
    assert all(r[3] > 0 for r in res)


def test_sweep_point_dealing():
    from paper_1012_4382_b200.sweep import shard_points, temperature_lambda_grid
    pts = temperature_lambda_grid()
    assert len(pts) == 64
    dealt = [shard_points(pts, r, 8) for r in range(8)]
    assert sorted(i for d in dealt for i, _ in d) == list(range(64))
    assert all(len(d) == 8 for d in dealt)


def _sweep_worker(rank, world, port, out_q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1012_4382_b200.sweep import run_sweep
    pts = list(range(11))
    res = run_sweep(pts, lambda p: (p, p * p, rank), workers=2, dist=dist)
    out_q.put((rank, res))
    dist.destroy_process_group()


def test_gloo_sweep_gathers_in_point_order():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sweep_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[1] is None
    assert [r[:2] for r in res[0]] == [(p, p * p) for p in range(11)]
    assert {r[2] for r in res[0]} == {0, 1}       # both ranks contributed

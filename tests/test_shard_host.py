"""Sharding host logic on CPU: halo plans from the link tables, and the halo
exchange protocol over torch.distributed (gloo, world_size 2) reproducing the
unsharded right-hand side bit for bit with the C oracle."""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1012_4382_b200.shard import (TILE, cross_halo_plan, device_tables_from_reference,
                                        halo_plan, shard_ranges, stage_output_buffer)


def lex_perm(indices):
    """device (pure lexicographic) position of every reference position"""
    order = np.lexsort(indices.T[::-1])
    perm = np.empty(len(order), np.int64)
    perm[order] = np.arange(len(order))
    return perm


def test_shard_ranges_cover_and_balance():
    r = shard_ranges(9993, 8)
    assert r[0][0] == 0 and sum(c for _, c in r) == 9993
    assert all(r[i][0] + r[i][1] == r[i + 1][0] for i in range(7))
    assert max(c for _, c in r) - min(c for _, c in r) <= 1
    with pytest.raises(ValueError):
        shard_ranges(3, 4)


@pytest.mark.parametrize("modes,n_max,shards", [(14, 3, 2), (14, 4, 5), (7, 6, 3)])
def test_halo_plan_is_complete_and_minimal(modes, n_max, shards):
    ind, _, plus, minus = orc.enumerate_hierarchy(modes, n_max)
    perm = lex_perm(ind)
    assert perm[0] == 0
    pd, md = device_tables_from_reference(plus, minus, perm)
    plan = halo_plan(pd, md, shards)
    n_tiles = (len(ind) + TILE - 1) // TILE
    for q, (b, c) in enumerate(plan.ranges):
        have = set(range(b, b + c))
        halo = set()
        for owner, first, cnt in plan.recv[q]:
            ob, oc = plan.ranges[owner]
            assert ob <= first and first + cnt <= ob + oc
            halo |= set(range(first, first + cnt))
        lo, hi = b * TILE, min((b + c) * TILE, len(ind))
        links = np.concatenate([pd[lo:hi].ravel(), md[lo:hi].ravel()])
        need = set((links[links >= 0] // TILE).tolist())
        assert need <= have | halo            # complete
        assert halo <= need and not (halo & have)  # minimal
        assert all(0 <= t < n_tiles for t in halo)
    sends = sorted((o, q, f, c) for q in range(shards) for o, f, c in plan.recv[q])
    assert sends == sorted((o, q, f, c) for o in range(shards) for q, f, c in plan.send[o])


@pytest.mark.parametrize("modes,kp1,n_max,shards", [(14, 2, 3, 2), (14, 2, 4, 5), (7, 1, 6, 3)])
def test_cross_halo_plan_is_complete_and_minimal(modes, kp1, n_max, shards):
    ind, _, plus, minus = orc.enumerate_hierarchy(modes, n_max)
    perm = lex_perm(ind)
    pd, md = device_tables_from_reference(plus, minus, perm)
    plan = cross_halo_plan(pd, md, shards, kp1, 7)
    for q, (b, c) in enumerate(plan.ranges):
        lo, hi = b * TILE, min((b + c) * TILE, len(ind))
        need = set()
        for m in range(modes):
            for t in np.concatenate([pd[lo:hi, m], md[lo:hi, m]]):
                if t >= 0 and not (b * TILE <= t < (b + c) * TILE):
                    need.add((int(t), m // kp1))
        got = set()
        for owner, pos, site in plan.recv[q]:
            ob, oc = plan.ranges[owner]
            assert np.all((pos >= ob * TILE) & (pos < (ob + oc) * TILE))
            assert np.all(np.diff(pos.astype(np.int64) * 16 + site) > 0)   # sorted, unique
            got |= set(zip(pos.tolist(), site.tolist()))
        assert got == need                      # complete and minimal
    pairs = sorted((o, q, len(p)) for q in range(shards) for o, p, _ in plan.recv[q])
    assert pairs == sorted((o, q, len(p)) for o in range(shards) for q, p, _ in plan.send[o])


def test_stage_buffers():
    assert [stage_output_buffer(s) for s in (1, 2, 3, 4)] == [1, 2, 3, 0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1012_4382_b200 as xf
    fmo = xf.build_fmo_system()
    bath = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
    rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
    pb = orc.Problem(fmo, bath, rates, 3, 1)
    perm = lex_perm(pb.indices)
    pd, md = device_tables_from_reference(pb.plus, pb.minus, perm)
    plan = halo_plan(pd, md, world)
    rng = np.random.default_rng(11)
    full = rng.standard_normal((pb.n_tot, 7, 7)) + 1j * rng.standard_normal((pb.n_tot, 7, 7))
    n_pad = ((pb.n_tot + TILE - 1) // TILE) * TILE
    dev = np.zeros((n_pad, 7, 7), complex)
    dev[perm] = full                       # device-order copy of the global state
    b, c = plan.ranges[rank]
    local = np.zeros_like(dev)             # this rank knows only its own tiles ...
    local[b * TILE:(b + c) * TILE] = dev[b * TILE:(b + c) * TILE]
    # ... plus the halo it receives from the owners (the transport of hb_exchange)
    reqs = []
    for dst, first, cnt in plan.send[rank]:
        t = torch.from_numpy(local[first * TILE:(first + cnt) * TILE].view(np.float64).copy())
        reqs.append(dist.isend(t, dst))
    for owner, first, cnt in plan.recv[rank]:
        t = torch.empty((cnt * TILE, 7, 7 * 2), dtype=torch.float64)
        dist.recv(t, owner)
        local[first * TILE:(first + cnt) * TILE] = t.numpy().view(np.complex128)
    for r in reqs:
        r.wait()
    rhs_local = pb.rhs(local[perm])        # oracle RHS on what this rank holds
    rhs_full = pb.rhs(full)
    mine = [k for k in range(pb.n_tot) if b * TILE <= perm[k] < (b + c) * TILE]
    ok = np.array_equal(rhs_local[mine], rhs_full[mine])
    out_q.put((rank, ok, len(mine), plan.halo_tiles(rank)))
    dist.destroy_process_group()


def _cross_worker(rank, world, port, out_q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1012_4382_b200 as xf
    fmo = xf.build_fmo_system()
    bath = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
    rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
    pb = orc.Problem(fmo, bath, rates, 3, 1)
    perm = lex_perm(pb.indices)
    pd, md = device_tables_from_reference(pb.plus, pb.minus, perm)
    plan = cross_halo_plan(pd, md, world, 2, 7)
    rng = np.random.default_rng(12)
    full = rng.standard_normal((pb.n_tot, 7, 7)) + 1j * rng.standard_normal((pb.n_tot, 7, 7))
    full = full + full.conj().transpose(0, 2, 1)          # Hermitian, like every ADO
    n_pad = ((pb.n_tot + TILE - 1) // TILE) * TILE
    dev = np.zeros((n_pad, 7, 7), complex)
    dev[perm] = full
    b, c = plan.ranges[rank]
    local = np.full_like(dev, np.nan)      # everything this rank does not own: unknown
    local[b * TILE:(b + c) * TILE] = dev[b * TILE:(b + c) * TILE]

    def cross(m, s):  # row and column s of each matrix: the 2d-1 shipped elements
        return np.concatenate([m[:, s, :], m[:, :, s]], axis=1)

    reqs = []
    for dst, pos, site in plan.send[rank]:
        payload = np.stack([cross(local[pos[i]:pos[i] + 1], site[i])[0] for i in range(len(pos))])
        reqs.append(dist.isend(torch.from_numpy(payload.view(np.float64).copy()), dst))
    for owner, pos, site in plan.recv[rank]:
        t = torch.empty((len(pos), 14, 2), dtype=torch.float64)
        dist.recv(t, owner)
        got = t.numpy().view(np.complex128)[..., 0]
        for i in range(len(pos)):
            local[pos[i], site[i], :] = got[i, :7]
            local[pos[i], :, site[i]] = got[i, 7:]
    for r in reqs:
        r.wait()
    rhs_local = pb.rhs(local[perm])
    rhs_full = pb.rhs(full)
    mine = [k for k in range(pb.n_tot) if b * TILE <= perm[k] < (b + c) * TILE]
    ok = np.array_equal(rhs_local[mine], rhs_full[mine])
    out_q.put((rank, ok, len(mine), plan.entries(rank)))
    dist.destroy_process_group()


def test_gloo_cross_halo_exchange_reproduces_unsharded_rhs():
    """only the crosses are shipped; the rest of every halo ADO is NaN here, so
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


def test_gloo_halo_exchange_reproduces_unsharded_rhs():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
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

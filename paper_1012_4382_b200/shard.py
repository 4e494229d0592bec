"""Sharded propagation of ONE hierarchy over several GPUs.

The device order is pure lexicographic (csrc/hb_graph.cu), so contiguous tile
ranges are the natural partition.  Each shard owns a range of tiles (32 ADOs)
and computes only those; before every stage it needs the neighbours of its
ADOs from the previous stage output -- the halo.  The halo plan is computed
once from the link tables:

  needed(q)  = tiles holding a raise/lower neighbour of an ADO owned by q,
               minus q's own tiles, grouped into runs of consecutive tiles
               per owner.

After stage s every owner sends those runs of the stage-s output buffer
(buffer s % 4: Y2, Y3, Y4, sigma) to the shards that need them.  Two transports:

* ``ShardedRun``      -- P shards inside this process (one or several local
  devices); the exchange is stream-ordered peer copies (hb_copy_tiles).  On a
  single GPU this is the bit-exact check of the partition and halo plan.
* ``NcclShardedRun``  -- one process per GPU (torchrun); grouped
  ncclSend/ncclRecv of the same tile runs (hb_exchange), NCCL over NVLink.

Both default to COMPRESSED halos (``exchange='crosses'``, cross_halo_plan): a
consumer reads from a halo ADO only the cross of the site it reaches it
through, so the plan ships (position, site) entries of 2d-1 planes instead of
whole tiles -- packed, grouped ncclSend/ncclRecv, unpacked (hb_halo_exchange),
or, for in-process shards on one device, copied in place (hb_halo_pull).

The root shard (tile 0 = ADO 0) integrates the sinks and records; sharded runs
use the t_end policy (a fixed number of steps, e.g. config 4: 1 ps).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .engine import BlockOperands, DeviceRun
from .hierarchy import enumerate_hierarchy

TILE = 32


def device_order_tables(modes: int, n_max: int, device: int = 0):
    """plus/minus in device (pure lexicographic) order from the reference-order
    tables and the permutation hb_graph_build exports."""
    g = enumerate_hierarchy(modes, n_max, device)
    return device_tables_from_reference(g.plus, g.minus, g.perm)


def device_tables_from_reference(plus, minus, perm):
    perm = np.asarray(perm, np.int64)
    n_tot = perm.shape[0]
    pd = np.empty_like(plus)
    md = np.empty_like(minus)
    pd[perm] = np.where(plus >= 0, perm[np.maximum(plus, 0)], plus)
    md[perm] = np.where(minus >= 0, perm[np.maximum(minus, 0)], minus)
    assert pd.shape[0] == n_tot
    return pd, md


def shard_ranges(n_tiles: int, n_shards: int):
    """Contiguous, balanced tile ranges [(begin, count)]."""
    if not 1 <= n_shards <= n_tiles:
        raise ValueError(f"cannot split {n_tiles} tiles into {n_shards} shards")
    bounds = np.linspace(0, n_tiles, n_shards + 1).round().astype(int)
    return [(int(bounds[i]), int(bounds[i + 1] - bounds[i])) for i in range(n_shards)]


def _runs(tiles):
    """sorted unique tiles -> [(first, count)] of consecutive runs"""
    out = []
    for t in tiles:
        if out and out[-1][0] + out[-1][1] == t:
            out[-1][1] += 1
        else:
            out.append([int(t), 1])
    return [(a, b) for a, b in out]


@dataclass
class HaloPlan:
    ranges: list          # [(begin, count)] per shard
    recv: list            # recv[q] = [(owner, first, count)]
    send: list            # send[r] = [(dest, first, count)]

    def halo_tiles(self, q: int) -> int:
        return sum(c for _, _, c in self.recv[q])


def halo_plan(plus_dev: np.ndarray, minus_dev: np.ndarray, n_shards: int) -> HaloPlan:
    n_tot = plus_dev.shape[0]
    n_tiles = (n_tot + TILE - 1) // TILE
    ranges = shard_ranges(n_tiles, n_shards)
    owner_of_tile = np.empty(n_tiles, np.int64)
    for r, (b, c) in enumerate(ranges):
        owner_of_tile[b:b + c] = r
    recv = [[] for _ in range(n_shards)]
    send = [[] for _ in range(n_shards)]
    for q, (b, c) in enumerate(ranges):
        lo, hi = b * TILE, min((b + c) * TILE, n_tot)
        links = np.concatenate([plus_dev[lo:hi].ravel(), minus_dev[lo:hi].ravel()])
        tiles = np.unique(links[links >= 0] // TILE)
        tiles = tiles[(tiles < b) | (tiles >= b + c)]
        for owner in np.unique(owner_of_tile[tiles]):
            for first, cnt in _runs(tiles[owner_of_tile[tiles] == owner]):
                recv[q].append((int(owner), first, cnt))
                send[int(owner)].append((q, first, cnt))
    return HaloPlan(ranges=ranges, recv=recv, send=send)


@dataclass
class CrossHaloPlan:
    """Compressed halos: per (consumer, owner) the (device position, site)
    entries whose cross (2d-1 planes) the consumer's kernels read."""
    ranges: list          # [(begin, count)] per shard
    recv: list            # recv[q] = [(owner, pos int32[], site int32[])]
    send: list            # send[o] = [(consumer, pos, site)] (the same arrays)
    n_planes_cross: int   # 2d - 1

    def entries(self, q: int) -> int:
        return sum(len(p) for _, p, _ in self.recv[q])

    def bytes_per_stage(self, q: int, elem: int = 8) -> int:
        return self.entries(q) * self.n_planes_cross * elem


def cross_halo_plan(plus_dev: np.ndarray, minus_dev: np.ndarray, n_shards: int, kp1: int,
                    d: int) -> CrossHaloPlan:
    """Mode m of the tables belongs to site m // kp1 (slot s = j(K+1) + k,
    identity site_of); a consumer reaching ADO t through mode m reads only the
    cross of that site (_kernels.py:41-57)."""
    n_tot, modes = plus_dev.shape
    n_tiles = (n_tot + TILE - 1) // TILE
    ranges = shard_ranges(n_tiles, n_shards)
    owner_of_tile = np.empty(n_tiles, np.int64)
    for r, (b, c) in enumerate(ranges):
        owner_of_tile[b:b + c] = r
    site_of_mode = np.arange(modes) // kp1
    recv = [[] for _ in range(n_shards)]
    send = [[] for _ in range(n_shards)]
    for q, (b, c) in enumerate(ranges):
        lo, hi = b * TILE, min((b + c) * TILE, n_tot)
        t = np.concatenate([plus_dev[lo:hi], minus_dev[lo:hi]]).astype(np.int64)
        s = np.broadcast_to(site_of_mode, t.shape)
        keep = (t >= 0) & ((t < b * TILE) | (t >= (b + c) * TILE))
        key = np.unique(t[keep] * 16 + s[keep])          # sorted by position, then site
        tt, ss = key // 16, key % 16
        own = owner_of_tile[tt // TILE]
        for owner in np.unique(own):
            sel = own == owner
            pos = np.ascontiguousarray(tt[sel], np.int32)
            site = np.ascontiguousarray(ss[sel], np.int32)
            recv[q].append((int(owner), pos, site))
            send[int(owner)].append((q, pos, site))
    return CrossHaloPlan(ranges=ranges, recv=recv, send=send, n_planes_cross=2 * d - 1)


def _halo_set(run: DeviceRun, segments):
    """segments: [(peer, is_send, pos, site)] -> hb_halo_set"""
    i32 = lambda x: np.ascontiguousarray(x, np.int32)
    peer = i32([g[0] for g in segments] or [0])
    is_send = i32([g[1] for g in segments] or [0])
    count = i32([len(g[2]) for g in segments] or [0])
    pos = i32(np.concatenate([g[2] for g in segments]) if segments else [0])
    site = i32(np.concatenate([g[3] for g in segments]) if segments else [0])
    N.check(N.lib().hb_halo_set(run._h, len(segments), N.ptr(peer), N.ptr(is_send), N.ptr(count),
                                N.ptr(pos), N.ptr(site)), "hb_halo_set")


def stage_output_buffer(stage: int) -> int:
    """Buffer index written by a stage: 1 -> Y2 (1), 2 -> Y3 (2), 3 -> Y4 (3), 4 -> sigma (0)."""
    return stage % 4


class ShardedRun:
    """P shards in one process; exchange = stream-ordered peer copies."""

    def __init__(self, ops: BlockOperands, n_max: int, dt_fs: float, t_end_fs: float,
                 n_shards: int, devices=None, record_stride: int = 1,
                 record_matrices: bool = False, blowup_norm: float = 1e6,
                 exchange: str = "crosses", precision: str = "double"):
        devices = devices or [0] * n_shards
        if exchange not in ("crosses", "tiles"):
            raise ValueError("exchange must be 'crosses' or 'tiles'")
        if exchange == "crosses" and len(set(devices)) > 1:
            raise ValueError("in-process compressed halos need all shards on one device")
        pd, md = device_order_tables(ops.modes, n_max, devices[0])
        self.exchange = exchange
        self.plan = halo_plan(pd, md, n_shards)
        self.cross_plan = cross_halo_plan(pd, md, n_shards, ops.n_matsubara + 1, ops.d) \
            if exchange == "crosses" else None
        self.n_tot = pd.shape[0]
        self.runs = [DeviceRun(ops, n_max, dt_fs, t_end_fs=t_end_fs, record_stride=record_stride,
                               record_matrices=record_matrices, blowup_norm=blowup_norm,
                               device=devices[q], layout="hermitian", tile_range=rg,
                               precision=precision, ordering="lex")
                     for q, rg in enumerate(self.plan.ranges)]

    def set_rho0(self, rho0_block, sink_pops):
        for r in self.runs:
            r.set_rho0(rho0_block, sink_pops)
        if self.cross_plan is not None:
            for q, r in enumerate(self.runs):
                _halo_set(r, [(o, 0, p, s) for o, p, s in self.cross_plan.recv[q]])

    def _exchange(self, stage: int):
        buf = stage_output_buffer(stage)
        if self.cross_plan is not None:
            for q, recv in enumerate(self.cross_plan.recv):
                for seg, (owner, _, _) in enumerate(recv):
                    N.check(N.lib().hb_halo_pull(self.runs[q]._h, self.runs[owner]._h, buf, seg),
                            "hb_halo_pull")
            return
        for q, recv in enumerate(self.plan.recv):
            for owner, first, cnt in recv:
                N.check(N.lib().hb_copy_tiles(self.runs[q]._h, self.runs[owner]._h, buf, first, cnt),
                        "hb_copy_tiles")

    def run(self, max_steps: int = 10 ** 9):
        """Step until the root shard stops (t_end); returns the root's status."""
        status = C.c_int(0)
        step = C.c_int64(0)
        N.check(N.lib().hb_sync(self.runs[0]._h, C.byref(status), C.byref(step)), "hb_sync")
        n = 0
        while status.value == 0 and n < max_steps:
            for s in (1, 2, 3, 4):
                for r in self.runs:
                    N.check(N.lib().hb_run_stage(r._h, s), "hb_run_stage")
                self._exchange(s)
            n += 1
            N.check(N.lib().hb_sync(self.runs[0]._h, C.byref(status), C.byref(step)), "hb_sync")
        for r in self.runs[1:]:
            st = C.c_int(0)
            N.check(N.lib().hb_sync(r._h, C.byref(st), None), "hb_sync")
            if st.value == 3:
                status.value = 3
        self.steps = step.value
        return status.value

    def records(self):
        return self.runs[0].records()

    def close(self):
        for r in self.runs:
            r.close()


class NcclShardedRun:
    """One process per GPU (torch.distributed initialised); NCCL halo exchange."""

    def __init__(self, ops: BlockOperands, n_max: int, dt_fs: float, t_end_fs: float,
                 rank: int, world: int, device: int, dist, record_stride: int = 10 ** 9,
                 exchange: str = "crosses"):
        pd, md = device_order_tables(ops.modes, n_max, device)
        self.plan = halo_plan(pd, md, world)
        self.cross_plan = cross_halo_plan(pd, md, world, ops.n_matsubara + 1, ops.d) \
            if exchange == "crosses" else None
        self.rank, self.world = rank, world
        self.run_ = DeviceRun(ops, n_max, dt_fs, t_end_fs=t_end_fs, record_stride=record_stride,
                              device=device, layout="hermitian", tile_range=self.plan.ranges[rank],
                              ordering="lex")
        uid = C.create_string_buffer(128)
        if rank == 0:
            N.check(N.lib().hb_nccl_unique_id(uid), "hb_nccl_unique_id")
        obj = [bytes(uid.raw)]
        dist.broadcast_object_list(obj, src=0)
        N.check(N.lib().hb_nccl_init(self.run_._h, C.create_string_buffer(obj[0], 128), world, rank),
                "hb_nccl_init")
        ent = [(p, f, c, 0) for p, f, c in self.plan.recv[rank]] + \
              [(p, f, c, 1) for p, f, c in self.plan.send[rank]]
        self._ex = [np.ascontiguousarray([e[i] for e in ent] or [0], np.int32) for i in range(4)]
        self._n_ex = len(ent)

    def set_rho0(self, rho0_block, sink_pops):
        self.run_.set_rho0(rho0_block, sink_pops)
        if self.cross_plan is not None:
            cp, r = self.cross_plan, self.rank
            _halo_set(self.run_, [(o, 0, p, s) for o, p, s in cp.recv[r]] +
                                 [(c, 1, p, s) for c, p, s in cp.send[r]])

    def enqueue_step(self):
        L = N.lib()
        for s in (1, 2, 3, 4):
            N.check(L.hb_run_stage(self.run_._h, s), "hb_run_stage")
            if self.cross_plan is not None:
                N.check(L.hb_halo_exchange(self.run_._h, stage_output_buffer(s)),
                        "hb_halo_exchange")
            else:
                N.check(L.hb_exchange(self.run_._h, stage_output_buffer(s), self._n_ex,
                                      *(N.ptr(a) for a in self._ex)), "hb_exchange")

    def sync(self):
        st, step = C.c_int(0), C.c_int64(0)
        N.check(N.lib().hb_sync(self.run_._h, C.byref(st), C.byref(step)), "hb_sync")
        return st.value, step.value

    def close(self):
        self.run_.close()

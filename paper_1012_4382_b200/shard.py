"""Sharded propagation of ONE hierarchy over several GPUs (new --
the reference declares distribution a non-goal).

Partition.  The ADOs are split into contiguous ranges of the pure
lexicographic order (n -> n + e_m preserves it, so a range keeps most of its
neighbours: at N_max = 8, K = 1, P = 8 a shard needs 8.6 MB of crosses per stage
against 59 MB for ranges of the reference's tier-major order).  Inside a shard
the owned ADOs are renumbered: those below the top tier first, tier-major like
the reference order, then the top-tier ones in whole tiles -- tiles with no
raise links, which the production kernel gathers in paired-site rounds
(csrc/hb_mm4.cu) -- then halo slots for the neighbours owned elsewhere.  A shard's buffers hold only its owned and halo
slots (``ShardLayout``).

Halo.  A kernel reads, from a neighbour reached through mode m, only the cross
of site(m): the 2d-1 Hermitian-packed planes of row/column site(m)
(_kernels.py:41-57).  So a consumer's halo plan lists (neighbour, site)
entries, and after every stage the owners ship those crosses of the stage
output (pack, grouped ncclSend/ncclRecv, unpack into the halo slots).

Overlap.  The owned tiles are split into four launch groups -- send-only,
interior, send+halo, halo-only -- so that per stage the tiles others need are
computed first and their crosses travel on a second stream while the rest
computes, and only the tiles that read halo slots wait for the incoming halo
(csrc/hb_shard.cu).  Every 25th step the divergence max is all-reduced.

Transports: ``NcclShardedRun`` (one process per GPU, torchrun) and
``ShardedRun`` (P shards in this process on one GPU, device copies instead of
NCCL: the bit-exactness check of partition, numbering and halo plan).
The root shard (ADO 0) integrates the sinks and records; sharded runs use the
t_end policy.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .engine import BlockOperands, DeviceRun
from .hierarchy import enumerate_hierarchy

TILE = 32


def lex_order(indices: np.ndarray) -> np.ndarray:
    """Reference positions sorted lexicographically (first mode most significant)."""
    return np.lexsort(indices.T[::-1])


def shard_bounds(n_tot: int, n_shards: int) -> np.ndarray:
    """Balanced contiguous ranges [bounds[q], bounds[q+1]) of the lexicographic order."""
    if not 1 <= n_shards <= n_tot:
        raise ValueError(f"cannot split {n_tot} ADOs into {n_shards} shards")
    return np.linspace(0, n_tot, n_shards + 1).round().astype(np.int64)


def stage_output_buffer(stage: int) -> int:
    """Buffer index written by a stage: 1 -> Y2 (1), 2 -> Y3 (2), 3 -> Y4 (3), 4 -> sigma (0)."""
    return stage % 4


@dataclass
class ShardLayout:
    """One shard: local slot numbering, local tables, halo plan, launch groups."""
    rank: int
    n_shards: int
    n_local: int              # slots (multiple of 32): owned tiles, then halo tiles
    own_tiles: int
    top_tile: int             # first owned tile of top-tier ADOs (own_tiles if none)
    root: bool                # slot 0 holds ADO 0
    local2ref: np.ndarray     # (n_local,) reference position of every slot, -1 = padding
    plus: np.ndarray          # (n_local, modes) local raise links, -1 = none
    minus: np.ndarray         # (n_local, modes) local lower links, -2 = none
    nvec: np.ndarray          # (n_local, modes) uint8
    recv: list = field(default_factory=list)   # [(owner, local halo slots, sites)]
    send: list = field(default_factory=list)   # [(consumer, local owned slots, sites)]
    groups: list = field(default_factory=list)  # 4 arrays of owned tiles

    @property
    def n_owned(self) -> int:
        return int(np.count_nonzero(self.local2ref[: self.own_tiles * TILE] >= 0))

    @property
    def n_halo(self) -> int:
        return int(np.count_nonzero(self.local2ref[self.own_tiles * TILE:] >= 0))

    def halo_entries(self) -> int:
        return sum(len(p) for _, p, _ in self.recv)

    def halo_bytes_per_stage(self, d: int = 7, elem: int = 8) -> int:
        return self.halo_entries() * (2 * d - 1) * elem


def build_shards(indices, tiers, plus, minus, n_shards: int, kp1: int, n_max: int):
    """Every shard's ShardLayout from the reference-order tables (hierarchy.py
    order, sentinels -1 / -2).  Mode m belongs to site m // kp1 (slot convention
    s = j (K+1) + k, identity site_of)."""
    n_tot, modes = plus.shape
    order = lex_order(indices)
    bounds = shard_bounds(n_tot, n_shards)
    owner = np.empty(n_tot, np.int64)
    for q in range(n_shards):
        owner[order[bounds[q]:bounds[q + 1]]] = q
    site_of_mode = (np.arange(modes) // kp1).astype(np.int64)
    layouts, halo_keys = [], []
    for q in range(n_shards):
        own = order[bounds[q]:bounds[q + 1]]
        top = tiers[own] == n_max
        # below the top tier: tier-major, lexicographic inside a tier (the
        # reference's own order restricted to the shard: the L2 window over these
        # tiles then holds the gather targets of the top tier); the top tier in
        # whole tiles after them
        low_part = own[~top]
        low_part = low_part[np.argsort(tiers[low_part], kind="stable")]
        top_part = own[top]
        a_tiles = -(-len(low_part) // TILE)
        own_tiles = a_tiles + -(-len(top_part) // TILE)
        # neighbours owned elsewhere, with the site they are reached through
        t = np.concatenate([plus[own], minus[own]]).astype(np.int64)
        s = np.broadcast_to(site_of_mode, t.shape)
        keep = t >= 0
        keep[keep] = owner[t[keep]] != q
        key = np.unique(t[keep] * 64 + s[keep])          # sorted by (position, site)
        halo_keys.append(key)
        halo_ado = np.unique(key // 64)
        n_local = (own_tiles + -(-len(halo_ado) // TILE)) * TILE
        local2ref = np.full(n_local, -1, np.int64)
        local2ref[:len(low_part)] = low_part
        local2ref[a_tiles * TILE:a_tiles * TILE + len(top_part)] = top_part
        local2ref[own_tiles * TILE:own_tiles * TILE + len(halo_ado)] = halo_ado
        layouts.append(ShardLayout(rank=q, n_shards=n_shards, n_local=n_local,
                                   own_tiles=own_tiles, top_tile=a_tiles if len(top_part) else own_tiles,
                                   root=bool(local2ref[0] == 0), local2ref=local2ref,
                                   plus=None, minus=None, nvec=None))
    for q, L in enumerate(layouts):
        g2l = np.full(n_tot, -1, np.int64)
        valid = L.local2ref >= 0
        g2l[L.local2ref[valid]] = np.nonzero(valid)[0]
        own_slots = L.own_tiles * TILE
        lp = np.full((L.n_local, modes), -1, np.int32)
        lm = np.full((L.n_local, modes), -2, np.int32)
        nv = np.zeros((L.n_local, modes), np.uint8)
        slots = np.nonzero(valid[:own_slots])[0]
        ref = L.local2ref[slots]
        pr, mr = plus[ref], minus[ref]
        lp[slots] = np.where(pr >= 0, g2l[np.maximum(pr, 0)], -1)
        lm[slots] = np.where(mr >= 0, g2l[np.maximum(mr, 0)], -2)
        nv[slots] = indices[ref]
        assert np.all((pr < 0) | (lp[slots] >= 0)) and np.all((mr < 0) | (lm[slots] >= 0)), \
            "halo plan incomplete"
        L.plus, L.minus, L.nvec = lp, lm, nv
        key = halo_keys[q]
        tt, ss = key // 64, key % 64
        own_t = owner[tt]
        for o in np.unique(own_t):
            sel = own_t == o
            L.recv.append((int(o), np.ascontiguousarray(g2l[tt[sel]], np.int32),
                           np.ascontiguousarray(ss[sel], np.int32), tt[sel]))
        # launch groups: X = tiles holding sent crosses, Y = tiles reading halo slots
        reads_halo = np.zeros(L.own_tiles, bool)
        links = np.concatenate([lp[:own_slots], lm[:own_slots]], axis=1)
        reads_halo |= np.any(links >= own_slots, axis=1).reshape(L.own_tiles, TILE).any(axis=1)
        L._reads_halo = reads_halo
    # sends: the consumer's entries (same order) at the owner's local slots
    for q, L in enumerate(layouts):
        for o, _, sites, refs in L.recv:
            W = layouts[o]
            valid = W.local2ref[: W.own_tiles * TILE] >= 0
            lookup = np.full(n_tot, -1, np.int64)
            lookup[W.local2ref[: W.own_tiles * TILE][valid]] = np.nonzero(valid)[0]
            pos = lookup[refs]
            assert np.all(pos >= 0)
            W.send.append((q, np.ascontiguousarray(pos, np.int32), sites))
    for L in layouts:
        L.recv = [(o, p, s) for o, p, s, _ in L.recv]
        sends = np.zeros(L.own_tiles, bool)
        for _, p, _ in L.send:
            sends[p // TILE] = True
        Y = L._reads_halo
        del L._reads_halo
        tiles = np.arange(L.own_tiles, dtype=np.int32)
        L.groups = [tiles[sends & ~Y], tiles[~sends & ~Y], tiles[sends & Y], tiles[~sends & Y]]
    return layouts


def _halo_set(run: DeviceRun, layout: ShardLayout):
    segs = [(o, 0, p, s) for o, p, s in layout.recv] + [(c, 1, p, s) for c, p, s in layout.send]
    i32 = lambda x: np.ascontiguousarray(x, np.int32)
    peer = i32([g[0] for g in segs] or [0])
    is_send = i32([g[1] for g in segs] or [0])
    count = i32([len(g[2]) for g in segs] or [0])
    pos = i32(np.concatenate([g[2] for g in segs]) if segs else [0])
    site = i32(np.concatenate([g[3] for g in segs]) if segs else [0])
    N.check(N.lib().hb_halo_set(run._h, len(segs), N.ptr(peer), N.ptr(is_send), N.ptr(count),
                                N.ptr(pos), N.ptr(site)), "hb_halo_set")


def t_end_steps(t_end_fs: float, dt_fs: float) -> int:
    """Steps of a t_end run: the smallest s with s dt >= t_end - 1e-9 (heom.py:359-361)."""
    s = max(0, int(math.floor((t_end_fs - 1e-9) / dt_fs)) - 2)
    while s * dt_fs < t_end_fs - 1e-9:
        s += 1
    return s


class _ShardBase:
    def _make_runs(self, ops, n_max, dt_fs, t_end_fs, layouts, devices, **kw):
        self.ops, self.n_max, self.dt = ops, n_max, dt_fs
        self.t_end = t_end_fs
        self.layouts = layouts
        self.runs = [DeviceRun(ops, n_max, dt_fs, t_end_fs=t_end_fs, device=dev, layout="hermitian",
                               shard=L, **kw) for L, dev in zip(layouts, devices)]

    def state(self, n_tot: int):
        """The global state (reference order) gathered from the shards' owned slots."""
        d = self.ops.d
        out = np.zeros((n_tot, d, d), np.complex128)
        for L, r in zip(self.layouts, self.runs):
            loc, _ = r.state(L.n_local)
            own = L.local2ref[: L.own_tiles * TILE]
            ok = own >= 0
            out[own[ok]] = loc[: L.own_tiles * TILE][ok]
        return out

    def close(self):
        for r in self.runs:
            r.close()


class ShardedRun(_ShardBase):
    """P shards in this process on one GPU (hb_shard_steps_local)."""

    def __init__(self, ops: BlockOperands, n_max: int, dt_fs: float, t_end_fs: float,
                 n_shards: int, device: int = 0, record_stride: int = 1,
                 record_matrices: bool = False, blowup_norm: float = 1e6,
                 precision: str = "double"):
        g = enumerate_hierarchy(ops.modes, n_max, device)
        layouts = build_shards(g.indices, g.tiers, g.plus, g.minus, n_shards,
                               ops.n_matsubara + 1, n_max)
        self._make_runs(ops, n_max, dt_fs, t_end_fs, layouts, [device] * n_shards,
                        record_stride=record_stride, record_matrices=record_matrices,
                        blowup_norm=blowup_norm, precision=precision)
        self.root = next(i for i, L in enumerate(layouts) if L.root)

    def set_rho0(self, rho0_block, sink_pops):
        for r, L in zip(self.runs, self.layouts):
            r.set_rho0(rho0_block, sink_pops)
            _halo_set(r, L)

    def steps(self, n: int) -> None:
        arr = (C.c_void_p * len(self.runs))(*[r._h for r in self.runs])
        N.check(N.lib().hb_shard_steps_local(arr, len(self.runs), int(n), None),
                "hb_shard_steps_local")

    def statuses(self):
        out = []
        for r in self.runs:
            st, step = C.c_int(0), C.c_int64(0)
            N.check(N.lib().hb_sync(r._h, C.byref(st), C.byref(step)), "hb_sync")
            out.append((st.value, step.value))
        return out

    def run(self, chunk: int = 25) -> int:
        """Step to t_end; stops early if any shard diverged.  Returns the root's
        status (1 = t_end, 3 = diverged)."""
        total = t_end_steps(self.t_end, self.dt)
        done = 0
        while done < total:
            n = min(chunk, total - done)
            self.steps(n)
            done += n
            st = self.statuses()
            if any(s == 3 for s, _ in st):
                return 3
        st = self.statuses()
        return 3 if any(s == 3 for s, _ in st) else st[self.root][0]

    def records(self):
        return self.runs[self.root].records()

    def sigma0(self):
        return self.runs[self.root].sigma0()


class NcclShardedRun(_ShardBase):
    """One process per GPU (torch.distributed initialised); NCCL halo exchange,
    overlapped with the interior tiles (hb_shard_steps)."""

    def __init__(self, ops: BlockOperands, n_max: int, dt_fs: float, t_end_fs: float,
                 rank: int, world: int, device: int, dist, record_stride: int = 10 ** 9):
        g = enumerate_hierarchy(ops.modes, n_max, device)
        layouts = build_shards(g.indices, g.tiers, g.plus, g.minus, world,
                               ops.n_matsubara + 1, n_max)
        self.rank, self.world, self.dist = rank, world, dist
        self.layout = layouts[rank]
        self._make_runs(ops, n_max, dt_fs, t_end_fs, [self.layout], [device],
                        record_stride=record_stride)
        self.layouts_all = layouts
        self.layouts = [self.layout]
        self.run_ = self.runs[0]
        uid = C.create_string_buffer(128)
        if rank == 0:
            N.check(N.lib().hb_nccl_unique_id(uid), "hb_nccl_unique_id")
        obj = [bytes(uid.raw)]
        dist.broadcast_object_list(obj, src=0)
        N.check(N.lib().hb_nccl_init(self.run_._h, C.create_string_buffer(obj[0], 128), world,
                                     rank), "hb_nccl_init")

    def set_rho0(self, rho0_block, sink_pops):
        self.run_.set_rho0(rho0_block, sink_pops)
        _halo_set(self.run_, self.layout)

    def steps(self, n: int, timed: bool = False):
        ms = C.c_double(0.0)
        N.check(N.lib().hb_shard_steps(self.run_._h, int(n), C.byref(ms) if timed else None),
                "hb_shard_steps")
        return ms.value if timed else None

    def time_steps(self, n: int) -> float:
        return self.steps(n, timed=True)

    def sync(self):
        """(status, step) of this shard, with the status all-reduced (MAX) over
        the ranks: any diverged shard stops all."""
        st, step = C.c_int(0), C.c_int64(0)
        N.check(N.lib().hb_sync(self.run_._h, C.byref(st), C.byref(step)), "hb_sync")
        import torch
        t = torch.tensor([st.value], dtype=torch.int64)
        if self.dist.get_backend() == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return int(t.item()), step.value

    def run(self, chunk: int = 25) -> int:
        total = t_end_steps(self.t_end, self.dt)
        done = 0
        while done < total:
            n = min(chunk, total - done)
            self.steps(n)
            done += n
            st, _ = self.sync()
            if st == 3:
                return 3
        return self.sync()[0]

    def launch_count(self) -> int:
        self.sync()  # the device-counted step kernels are read at a synchronisation
        return self.run_.launch_count()

    def describe(self) -> dict:
        L = self.layout
        return {"owned_ados_rank0": self.layouts_all[0].n_owned,
                "halo_ados_max": max(x.n_halo for x in self.layouts_all),
                "halo_bytes_per_stage_max": max(x.halo_bytes_per_stage() for x in self.layouts_all),
                "slots_rank0": self.layouts_all[0].n_local,
                "groups_rank0": [int(len(g)) for g in self.layouts_all[0].groups],
                "rank_groups": [int(len(g)) for g in L.groups]}

"""Hierarchy topology: multi-indices and raise/lower neighbour tables.

Drop-in for the reference hierarchy.py (enumerate_hierarchy :59-105,
hierarchy_size :27-29, index_of :108-114, sentinels :18-21).  The tables are
built on the GPU by ``hb_graph_build`` (csrc/hb_graph.cu: every thread ranks its
multi-index with a binomial table) and returned in the reference order
(tier-major, lexicographic within a tier), bit-identical to the reference.
The tuple lookup is a combinatorial rank instead of a dict.
"""

from __future__ import annotations

import math
from collections.abc import Mapping
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

#: raise-neighbour sentinel: n + e_m would exceed the truncation tier
TRUNCATED = -1
#: lower-neighbour sentinel: n_m = 0
ABSENT = -2

_MAX_INDEX = np.iinfo(np.int32).max


def hierarchy_size(n_sites: int, n_max: int) -> int:
    """C(n_sites + n_max, n_sites): multi-indices with tier <= n_max."""
    return math.comb(n_sites + n_max, n_sites)


class GradedLookup(Mapping):
    """tuple -> reference position, computed (graded lexicographic rank)."""

    def __init__(self, n_sites: int, n_max: int, indices: np.ndarray):
        self.n_sites, self.n_max, self._indices = n_sites, n_max, indices

    def _rank(self, key):
        M = self.n_sites
        if len(key) != M or any(v < 0 for v in key):
            raise KeyError(key)
        t = sum(key)
        if t > self.n_max:
            raise KeyError(key)
        r = hierarchy_size(M, t - 1) if t > 0 else 0
        rem = t
        for i in range(M - 1):
            parts = M - i - 1
            for v in range(key[i]):
                r += math.comb(rem - v + parts - 1, parts - 1)
            rem -= key[i]
        return r

    def __getitem__(self, key):
        return self._rank(tuple(int(v) for v in key))

    def __contains__(self, key):
        try:
            self._rank(tuple(int(v) for v in key))
            return True
        except (KeyError, TypeError, ValueError):
            return False

    def __len__(self):
        return int(self._indices.shape[0])

    def __iter__(self):
        for row in self._indices:
            yield tuple(int(v) for v in row)


@dataclass(frozen=True)
class HierarchyGraph:
    """Immutable truncated hierarchy (reference order) and its neighbour links."""

    n_sites: int
    n_max: int
    indices: np.ndarray
    tiers: np.ndarray
    plus: np.ndarray
    minus: np.ndarray
    lookup: Mapping = field(repr=False)
    #: device (pure-lexicographic) position of every reference position
    perm: np.ndarray = field(default=None, repr=False)

    @property
    def n_tot(self) -> int:
        return int(self.indices.shape[0])


def enumerate_hierarchy(n_sites: int, n_max: int, device: int = 0) -> HierarchyGraph:
    """All multi-indices with tier <= n_max and their neighbour links (GPU-built)."""
    if n_sites < 1:
        raise ValueError("need at least one site")
    if n_max < 0:
        raise ValueError("truncation tier must be >= 0")
    n_tot = hierarchy_size(n_sites, n_max)
    if n_tot > _MAX_INDEX:
        raise ValueError(f"hierarchy with {n_tot} indices exceeds the supported index range")
    N.require_device(device)
    indices = np.empty((n_tot, n_sites), np.int32)
    tiers = np.empty(n_tot, np.int32)
    plus = np.empty((n_tot, n_sites), np.int32)
    minus = np.empty((n_tot, n_sites), np.int32)
    perm = np.empty(n_tot, np.int32)
    rc = N.lib().hb_graph_build(n_sites, n_max, device, N.ptr(indices), N.ptr(tiers),
                                N.ptr(plus), N.ptr(minus), N.ptr(perm))
    N.check(rc, "hb_graph_build")
    for a in (indices, tiers, plus, minus, perm):
        a.setflags(write=False)
    return HierarchyGraph(n_sites=n_sites, n_max=n_max, indices=indices, tiers=tiers,
                          plus=plus, minus=minus, lookup=GradedLookup(n_sites, n_max, indices),
                          perm=perm)


def index_of(graph: HierarchyGraph, multi_index) -> int:
    """Position of a multi-index; KeyError outside the truncated set."""
    key = tuple(int(n) for n in multi_index)
    try:
        return graph.lookup[key]
    except KeyError:
        raise KeyError(f"multi-index {key} not in hierarchy (n_max={graph.n_max})") from None

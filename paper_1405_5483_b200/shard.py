"""Text sharding across ranks (one process per GPU).

The search partitions by text position with no data-path exchange
(SURVEY.md §8e): rank g owns the start offsets [a_g, a_{g+1}) and searches
the read span [a_g, min(n, a_{g+1} + maxlen - 1)) as a standalone text, so
every occurrence that starts in its range is found exactly (an occurrence
never needs bytes before its own start).  Occurrences that start at or
after a_{g+1} belong to the next rank and are dropped.  Each rank's list is
already sorted by (offset, pattern_index) and the ranges are disjoint and
ordered, so the one collective is a gather that concatenates in rank order.

Masks, maps and pattern tables are replicated: each rank builds its own
engine from the same pattern set.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

ALIGN = 4096  # ownership boundaries are page aligned: device sub-pointers stay 16 B aligned


def ownership(n: int, world: int, align: int = ALIGN) -> List[int]:
    """Boundaries a_0=0 <= a_1 <= ... <= a_world=n, interior ones multiples of `align`."""
    if world < 1:
        raise ValueError("world must be >= 1")
    per = -(-n // world)
    per = -(-per // align) * align if n > align * world else per
    b = [min(n, g * per) for g in range(world)] + [n]
    return b


def read_span(n: int, bounds: Sequence[int], rank: int, maxlen: int) -> Tuple[int, int]:
    """Bytes rank `rank` must read: its owned starts plus maxlen-1 of halo."""
    lo, own_end = bounds[rank], bounds[rank + 1]
    if own_end <= lo:
        return lo, lo
    return lo, min(n, own_end + maxlen - 1)


def clip(offs: np.ndarray, pids: np.ndarray, lo: int, own_end: int) -> Tuple[np.ndarray, np.ndarray]:
    """Local (span-relative) results -> global offsets owned by this rank."""
    keep = offs < np.uint64(own_end - lo)
    return offs[keep] + np.uint64(lo), pids[keep]


def gather(offs: np.ndarray, pids: np.ndarray, world: int, rank: int, dst: int = 0, group=None):
    """The one exchange: concatenate every rank's (sorted, disjoint) list on
    `dst` in rank order.  Returns the global arrays on dst, None elsewhere."""
    if world == 1:
        return offs, pids
    import torch.distributed as dist
    objs: Optional[list] = [None] * world if rank == dst else None
    dist.gather_object((offs, pids), objs, dst=dst, group=group)
    if rank != dst:
        return None
    o = np.concatenate([x[0] for x in objs]) if objs else np.zeros(0, np.uint64)
    p = np.concatenate([x[1] for x in objs]) if objs else np.zeros(0, np.uint32)
    return o.astype(np.uint64), p.astype(np.uint32)


def sharded_search(search: Callable[[int, int], Tuple[np.ndarray, np.ndarray]], n: int, maxlen: int,
                   world: int, rank: int, group=None, dst: int = 0):
    """Run `search(lo, hi)` (sorted span-relative (offsets, pattern ids) of
    text[lo:hi]) on this rank's span and gather the global result on dst."""
    bounds = ownership(n, world)
    lo, hi = read_span(n, bounds, rank, maxlen)
    if hi > lo:
        o, p = search(lo, hi)
        o, p = clip(np.asarray(o, dtype=np.uint64), np.asarray(p, dtype=np.uint32), lo, bounds[rank + 1])
    else:
        o, p = np.zeros(0, np.uint64), np.zeros(0, np.uint32)
    return gather(o, p, world, rank, dst=dst, group=group)


def engine_span_search(engine, d_text_ptr: int, keep=None):
    """`search` callable for sharded_search over device-resident text: the
    span is searched in place through mag_prepare_device_text."""

    def run(lo: int, hi: int):
        prep = engine.prepare_device(d_text_ptr + lo, hi - lo, keep=keep)
        try:
            m = engine.search_prepared(prep)
            try:
                return m.arrays()
            finally:
                m.close()
        finally:
            prep.close()

    return run

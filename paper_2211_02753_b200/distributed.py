"""Row-sharded multi-GPU execution: one process per GPU, NCCL over NVLink.

Scans, filters and aggregations shard row-wise (each rank holds a contiguous
slice of every base table).  Inside :func:`sharded`, the exact group-by and
global aggregates compute dense *partials* on the local shard with the fused
kernel and merge them with NCCL all-reduces before finalising:

* key ranges of plain integer keys: all-reduce MIN / MAX (so every rank
  agrees on the dense slot layout);
* per-slot counts (int64) and integer sums: all-reduce SUM (exact);
* float64 sums: all-reduce SUM.

Averages and the occupied-group compaction are computed after the merge, so
results equal the single-GPU result (float sums up to summation order).
The reference has no distribution at all.
"""

from __future__ import annotations

import threading
from contextlib import contextmanager
from typing import Optional

import torch
import torch.distributed as dist

_TLS = threading.local()


def current_group():
    """The process group of the enclosing :func:`sharded` block, or None."""
    return getattr(_TLS, "group", None)


@contextmanager
def sharded(group=None):
    """Run queries on the local shard and merge aggregates across ``group``
    (default: the world group when torch.distributed is initialised)."""
    if group is None and dist.is_available() and dist.is_initialized():
        group = dist.group.WORLD
    prev = getattr(_TLS, "group", None)
    _TLS.group = group
    try:
        yield group
    finally:
        _TLS.group = prev


def world_size(group) -> int:
    return 1 if group is None else dist.get_world_size(group)


def allreduce_ranges(lo: torch.Tensor, hi: torch.Tensor, group) -> tuple[torch.Tensor, torch.Tensor]:
    """Global [min, max] of per-rank key ranges (empty shards hold
    (INT64_MAX, INT64_MIN), the identities of MIN / MAX)."""
    if world_size(group) > 1:
        dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    return lo, hi


def allreduce_partials(counts: torch.Tensor, sums_raw: torch.Tensor, float_rows: list[int],
                       group) -> None:
    """In-place SUM of dense partial aggregates across ranks.

    ``counts``: int64 [slots].  ``sums_raw``: int64 [naggs, slots] holding the
    raw 8-byte results; rows listed in ``float_rows`` are float64 bit
    patterns, the others int64 (counts / integer sums, wrap-around).
    """
    if world_size(group) <= 1:
        return
    nrows = sums_raw.shape[0]
    int_rows = [r for r in range(nrows) if r not in float_rows]
    ints = torch.cat([counts.reshape(1, -1), sums_raw[int_rows]], dim=0) if int_rows else counts.reshape(1, -1).clone()
    dist.all_reduce(ints, op=dist.ReduceOp.SUM, group=group)
    counts.copy_(ints[0])
    for j, r in enumerate(int_rows):
        sums_raw[r].copy_(ints[1 + j])
    if float_rows:
        floats = sums_raw[float_rows].contiguous().view(torch.float64).clone()
        dist.all_reduce(floats, op=dist.ReduceOp.SUM, group=group)
        for j, r in enumerate(float_rows):
            sums_raw[r].copy_(floats[j].view(torch.int64))


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row range of ``rank`` (sizes differ by at most one row)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)

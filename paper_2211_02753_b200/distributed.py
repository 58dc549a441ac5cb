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

import os
import threading
from contextlib import contextmanager

import torch
import torch.distributed as dist

from . import hostread

_TLS = threading.local()

# TDP_FORCE_COLLECTIVES=1: a one-rank group still takes the sharded code path
# (partials, NCCL all-reduce / all-to-all over a real one-rank communicator) --
# how the collective path is exercised on a single-GPU host.
def _force() -> bool:
    return os.environ.get("TDP_FORCE_COLLECTIVES") == "1"


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


def is_sharded(group) -> bool:
    """Rows of ``group``'s relations are split across ranks (merge needed)."""
    return group is not None and (dist.get_world_size(group) > 1 or _force())


@contextmanager
def local():
    """Suspend the enclosing :func:`sharded` scope: the computation inside
    sees one rank's data as the whole (an aggregate over a relation every
    rank already holds in full must not be merged again)."""
    prev = getattr(_TLS, "group", None)
    _TLS.group = None
    try:
        yield
    finally:
        _TLS.group = prev


# Collectives: NCCL on device tensors.  A gloo group (CPU tests, or several
# ranks sharing one GPU in the test harness) gets host-staged copies.
def _host_staged(group) -> bool:
    return dist.get_backend(group) == "gloo"


def _all_reduce(t: torch.Tensor, op, group) -> None:
    if t.is_cuda and _host_staged(group):
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)


def _all_to_all_single(out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits, group) -> None:
    if inp.is_cuda and _host_staged(group):
        h = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(h, inp.cpu(), out_splits, in_splits, group=group)
        out.copy_(h)
    else:
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)


def _all_gather(parts: list, t: torch.Tensor, group) -> None:
    if t.is_cuda and _host_staged(group):
        hs = [torch.empty(p.shape, dtype=p.dtype) for p in parts]
        dist.all_gather(hs, t.cpu(), group=group)
        for p, h in zip(parts, hs):
            p.copy_(h)
    else:
        dist.all_gather(parts, t, group=group)


class _AllReduceSum(torch.autograd.Function):
    """Sum of per-rank partial grids across ranks, differentiable: everything
    downstream (loss, its gradient) is computed from the reduced grid, so the
    upstream gradient is the same on every rank and is also the gradient of
    each rank's partial; the parameter gradients that result are per-rank
    partial sums (reduced by the trainer, training.train_step)."""

    @staticmethod
    def forward(ctx, t: torch.Tensor, group) -> torch.Tensor:
        out = t.detach().clone()
        _all_reduce(out, dist.ReduceOp.SUM, group)
        return out

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        return g, None


def allreduce_sum(t: torch.Tensor, group) -> torch.Tensor:
    """``t`` summed over the ranks of ``group`` (identity for one rank),
    keeping the autograd graph (soft group-by grids of a sharded LLP step)."""
    if not is_sharded(group):
        return t
    return _AllReduceSum.apply(t, group)


def allreduce_grads(grads, group) -> None:
    """In-place SUM of per-rank parameter gradients (data-parallel step)."""
    if not is_sharded(group):
        return
    for g in grads:
        if g is not None:
            _all_reduce(g, dist.ReduceOp.SUM, group)


def allreduce_ranges(lo: torch.Tensor, hi: torch.Tensor, group) -> tuple[torch.Tensor, torch.Tensor]:
    """Global [min, max] of per-rank key ranges (empty shards hold
    (INT64_MAX, INT64_MIN), the identities of MIN / MAX)."""
    if is_sharded(group):
        _all_reduce(lo, dist.ReduceOp.MIN, group)
        _all_reduce(hi, dist.ReduceOp.MAX, group)
    return lo, hi


def allreduce_partials(counts: torch.Tensor, sums_raw: torch.Tensor, float_rows: list[int],
                       group, count_rows: tuple = ()) -> None:
    """In-place SUM of dense partial aggregates across ranks.

    ``counts``: int64 [slots].  ``sums_raw``: int64 [naggs, slots] holding the
    raw 8-byte results; rows listed in ``float_rows`` are float64 bit
    patterns, the others int64 (counts / integer sums, wrap-around).  When
    every integer row is a count (``count_rows``), counts travel as float64
    (exact: a row count is far below 2^53) in the same all-reduce as the float
    sums -- one collective per query instead of two.
    """
    if not is_sharded(group):
        return
    nrows = sums_raw.shape[0]
    int_rows = [r for r in range(nrows) if r not in float_rows]
    # rows by slicing (no advanced indexing: a host index list would be a
    # pageable copy, which a CUDA-graph capture cannot contain)
    row = lambda r: sums_raw[r:r + 1]  # noqa: E731
    if all(r in count_rows for r in int_rows):
        merged = torch.cat([counts.reshape(1, -1).to(torch.float64)]
                           + [row(r).to(torch.float64) for r in int_rows]
                           + [row(r).view(torch.float64) for r in float_rows], dim=0)
        _all_reduce(merged, dist.ReduceOp.SUM, group)
        counts.copy_(merged[0].round().to(torch.int64))
        for j, r in enumerate(int_rows):
            sums_raw[r].copy_(merged[1 + j].round().to(torch.int64))
        for j, r in enumerate(float_rows):
            sums_raw[r].copy_(merged[1 + len(int_rows) + j].view(torch.int64))
        return
    ints = torch.cat([counts.reshape(1, -1)] + [row(r) for r in int_rows], dim=0)
    _all_reduce(ints, dist.ReduceOp.SUM, group)
    counts.copy_(ints[0])
    for j, r in enumerate(int_rows):
        sums_raw[r].copy_(ints[1 + j])
    if float_rows:
        floats = torch.cat([row(r) for r in float_rows], dim=0).view(torch.float64)
        _all_reduce(floats, dist.ReduceOp.SUM, group)
        for j, r in enumerate(float_rows):
            sums_raw[r].copy_(floats[j].view(torch.int64))


def key_destination(keys: list[torch.Tensor], world: int) -> torch.Tensor:
    """Owner rank of each row: a 64-bit mix of the key tuple, mod world.
    Equal key tuples always map to the same rank."""
    h = torch.zeros_like(keys[0], dtype=torch.int64)
    for k in keys:
        x = k.to(torch.int64) ^ (h * 31)
        # splitmix64 finaliser in two's-complement int64 arithmetic
        x = x ^ ((x >> 30) & 0x3FFFFFFFF)
        x = x * -4658895280553007687  # 0xbf58476d1ce4e5b9
        x = x ^ ((x >> 27) & 0x1FFFFFFFFF)
        x = x * -7723592293110705685  # 0x94d049bb133111eb
        h = x ^ ((x >> 31) & 0x1FFFFFFFF)
    return torch.remainder(h, world)


def exchange_rows(grouped: list[torch.Tensor], send_counts: torch.Tensor,
                  group) -> list[torch.Tensor]:
    """All-to-all repartition of rows (NCCL on the GPU host).

    ``grouped`` columns hold the local rows already ordered by destination
    rank (a stable sort of the destinations, done by the caller with the
    radix-sort kernel) and ``send_counts[r]`` is how many go to rank r.  Rows
    arrive grouped by source rank, each group in its original order, so the
    result is deterministic.
    """
    recv_counts = torch.empty_like(send_counts)
    _all_to_all_single(recv_counts, send_counts, None, None, group)
    # one host read of both split vectors (hostread: logged for graph replay,
    # checked on the device when replayed)
    both = hostread.read_ints(torch.cat([send_counts, recv_counts]))
    world = send_counts.numel()
    send, recv = both[:world], both[world:]
    out = []
    for col in grouped:
        dst = torch.empty((sum(recv),) + tuple(col.shape[1:]), dtype=col.dtype, device=col.device)
        _all_to_all_single(dst, col.contiguous(), recv, send, group)
        out.append(dst)
    return out


def allgather_rows(columns: list[torch.Tensor], group) -> list[torch.Tensor]:
    """Concatenate every rank's rows (rank order) on every rank."""
    world = world_size(group)
    if not is_sharded(group):
        return columns
    dev = columns[0].device
    n = torch.tensor([columns[0].shape[0]], dtype=torch.int64, device=dev)
    sizes = [torch.empty_like(n) for _ in range(world)]
    _all_gather(sizes, n, group)
    sizes = hostread.read_ints(torch.cat(sizes))
    m = max(sizes) if sizes else 0
    out = []
    for col in columns:
        pad = torch.zeros((m,) + tuple(col.shape[1:]), dtype=col.dtype, device=dev)
        pad[: col.shape[0]] = col
        parts = [torch.empty_like(pad) for _ in range(world)]
        _all_gather(parts, pad, group)
        out.append(torch.cat([p[:s] for p, s in zip(parts, sizes)]))
    return out


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row range of ``rank`` (sizes differ by at most one row)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)

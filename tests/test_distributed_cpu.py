"""CPU, world size 2 over gloo: the multi-GPU merge logic of distributed.py.

The GPU path computes dense partials with the fused kernel on each rank's row
shard and merges them with these collectives (NCCL on the GPU host).  Here
each rank builds its partials with the oracle and the merged result must equal
the single-process oracle over all rows.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_02753_b200.distributed import allreduce_partials, allreduce_ranges, shard_bounds


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _dense_partials(keys, vf, vi, lo, span):
    """Oracle dense partials over slots [0, span): counts, float sums, int sums."""
    slot = keys - lo
    counts = np.bincount(slot, minlength=span).astype(np.int64)
    fs = np.zeros(span)
    np.add.at(fs, slot, vf)
    is_ = np.zeros(span, dtype=np.int64)
    np.add.at(is_, slot, vi)
    return counts, fs, is_


def _worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    n = 10_001
    keys = rng.integers(5, 40, size=n)
    vf = rng.normal(size=n)
    vi = rng.integers(-100, 100, size=n)
    a, b = shard_bounds(n, rank, world)
    k, f, i = keys[a:b], vf[a:b], vi[a:b]
    lo_t = torch.tensor([k.min() if len(k) else np.iinfo(np.int64).max])
    hi_t = torch.tensor([k.max() if len(k) else np.iinfo(np.int64).min])
    lo_t, hi_t = allreduce_ranges(lo_t, hi_t, dist.group.WORLD)
    lo, hi = int(lo_t), int(hi_t)
    span = hi - lo + 1
    counts, fs, is_ = _dense_partials(k, f, i, lo, span)
    c_t = torch.from_numpy(counts)
    raw = torch.stack([torch.from_numpy(fs).view(torch.int64), torch.from_numpy(is_), c_t.clone()])
    # merged path: count rows travel with the float sums in one all-reduce
    c2 = torch.from_numpy(counts.copy())
    raw2 = torch.stack([torch.from_numpy(fs.copy()).view(torch.int64), c2.clone()])
    allreduce_partials(c2, raw2, [0], dist.group.WORLD, count_rows=(1,))
    allreduce_partials(c_t, raw, [0], dist.group.WORLD)
    if rank == 0:
        exp_c, exp_f, exp_i = _dense_partials(keys, vf, vi, keys.min(), keys.max() - keys.min() + 1)
        result["ok"] = (lo == keys.min() and hi == keys.max()
                        and np.array_equal(c_t.numpy(), exp_c)
                        and np.allclose(raw[0].view(torch.float64).numpy(), exp_f, rtol=1e-12)
                        and np.array_equal(raw[1].numpy(), exp_i)
                        and np.array_equal(raw[2].numpy(), exp_c)
                        and np.array_equal(c2.numpy(), exp_c)
                        and c2.dtype == torch.int64
                        and np.array_equal(raw2[1].numpy(), exp_c)
                        and np.allclose(raw2[0].view(torch.float64).numpy(), exp_f, rtol=1e-12))
    dist.destroy_process_group()


def test_allreduce_partials_world2():
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), result), nprocs=2, join=True)
    assert result.get("ok") is True


def _shuffle_worker(rank, world, port, result):
    """High-cardinality group-by across ranks: key_destination + all-to-all
    exchange + local group-by + all-gather + lexicographic order (the GPU
    path's steps; local sort / group-by done by the oracle here)."""
    from oracle import relational as orc
    from paper_2211_02753_b200.distributed import allgather_rows, exchange_rows, key_destination

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(1)
    n = 20_000
    k1 = rng.integers(-10**9, 10**9, size=n // 7)[rng.integers(0, n // 7, size=n)]
    k2 = rng.integers(0, 3, size=n)
    v = rng.normal(size=n)
    a, b = shard_bounds(n, rank, world)
    kk1, kk2, vv = (torch.from_numpy(x[a:b].copy()) for x in (k1, k2, v))
    dest = key_destination([kk1, kk2], world)
    order = torch.from_numpy(np.argsort(dest.numpy(), kind="stable"))
    counts = torch.from_numpy(np.bincount(dest.numpy(), minlength=world).astype(np.int64))
    rk1, rk2, rv = exchange_rows([t[order] for t in (kk1, kk2, vv)], counts, dist.group.WORLD)
    keys, aggs = orc.groupby_exact([rk1.numpy(), rk2.numpy()], [("sum", rv.numpy()), ("count", None)])
    g1, g2, gs, gc = allgather_rows([torch.from_numpy(x) for x in (*keys, *aggs)], dist.group.WORLD)
    o = np.lexsort((g2.numpy(), g1.numpy()))
    if rank == 0:
        ekeys, eaggs = orc.groupby_exact([k1, k2], [("sum", v), ("count", None)])
        result["ok"] = (np.array_equal(g1.numpy()[o], ekeys[0])
                        and np.array_equal(g2.numpy()[o], ekeys[1])
                        and np.array_equal(gc.numpy()[o], eaggs[1])
                        and np.allclose(gs.numpy()[o], eaggs[0], rtol=1e-12)
                        and int(counts.sum()) == b - a)
    dist.destroy_process_group()


def test_key_shuffle_group_by_world2():
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_shuffle_worker, args=(2, _free_port(), result), nprocs=2, join=True)
    assert result.get("ok") is True


def test_key_destination_is_a_function_of_the_key():
    from paper_2211_02753_b200.distributed import key_destination

    k = torch.tensor([5, -7, 5, 2**62, -7, 0])
    d = key_destination([k], 4)
    assert d.tolist()[0] == d.tolist()[2] and d.tolist()[1] == d.tolist()[4]
    assert d.min() >= 0 and d.max() < 4
    many = key_destination([torch.arange(100_000)], 8)
    counts = torch.bincount(many, minlength=8)
    assert counts.min() > 100_000 / 8 * 0.9  # spreads keys evenly


def test_shard_bounds_cover_rows():
    for n in (0, 1, 7, 10**6 + 3):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[r][1] == spans[r + 1][0] for r in range(w - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _grad_worker(rank, world, port, result):
    """allreduce_sum: forward = sum of the ranks' partials, backward = the
    upstream gradient on every rank; allreduce_grads sums the partials."""
    from paper_2211_02753_b200.distributed import allreduce_grads, allreduce_sum

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = torch.tensor([1.0, 2.0, 3.0], dtype=torch.float64) * (rank + 1)
    t.requires_grad_(True)
    out = allreduce_sum(t, dist.group.WORLD)
    w = torch.tensor([0.5, -1.0, 2.0], dtype=torch.float64)
    (out * w).sum().backward()
    g = [t.grad.clone()]
    allreduce_grads(g, dist.group.WORLD)
    if rank == 0:
        result["ok"] = (torch.equal(out.detach(), torch.tensor([3.0, 6.0, 9.0], dtype=torch.float64))
                        and torch.equal(t.grad, w) and torch.equal(g[0], 2 * w))
    dist.destroy_process_group()


def test_differentiable_allreduce_world2():
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_grad_worker, args=(2, _free_port(), result), nprocs=2, join=True)
    assert result.get("ok") is True

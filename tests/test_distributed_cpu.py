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
    allreduce_partials(c_t, raw, [0], dist.group.WORLD)
    if rank == 0:
        exp_c, exp_f, exp_i = _dense_partials(keys, vf, vi, keys.min(), keys.max() - keys.min() + 1)
        result["ok"] = (lo == keys.min() and hi == keys.max()
                        and np.array_equal(c_t.numpy(), exp_c)
                        and np.allclose(raw[0].view(torch.float64).numpy(), exp_f, rtol=1e-12)
                        and np.array_equal(raw[1].numpy(), exp_i)
                        and np.array_equal(raw[2].numpy(), exp_c))
    dist.destroy_process_group()


def test_allreduce_partials_world2():
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), result), nprocs=2, join=True)
    assert result.get("ok") is True


def test_shard_bounds_cover_rows():
    for n in (0, 1, 7, 10**6 + 3):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[r][1] == spans[r + 1][0] for r in range(w - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1

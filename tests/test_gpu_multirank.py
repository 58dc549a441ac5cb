"""GPU, 2 ranks on one device (gloo, host-staged collectives): the sharded
execution path with the real kernels.

Production multi-GPU runs use NCCL with one rank per GPU; this test drives the
same code (row-sharded fused aggregates + all-reduce merge, high-cardinality
group-by with key repartition + all-gather) on the single GPU available to the
test harness.  Results must equal the single-process oracle over all rows.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2211_02753_b200 as tq
    from oracle import relational as orc
    from oracle import tpch as otpch
    from paper_2211_02753_b200 import workloads as wl
    from paper_2211_02753_b200.distributed import shard_bounds, sharded

    ok = True
    # Q1 row-sharded: dense partials merged by all-reduce
    arrays = wl.lineitem_arrays(0.01, seed=4, rows=100_003)
    a, b = shard_bounds(100_003, rank, world)
    shard = {k: v[a:b] for k, v in arrays.items()}
    cat = tq.Catalog()
    cat.register("lineitem", wl.lineitem_table(shard))
    q = wl.compile_sql(wl.Q1_SQL, cat, wl.q1_registry())
    with sharded():
        res = q.run(cat)
    got = {n: c.values.numpy() for n, c in zip(res.schema.names, res.columns)}
    exp = otpch.q1(arrays)
    _c = bool(np.array_equal(got["rf"], exp["rf"]) and np.array_equal(got["count"], exp["count"]))
    if not _c:
        import sys
        print(f'rank {rank}: check at line 55 failed', file=sys.stderr, flush=True)
    ok &= _c
    _c = bool(all(np.allclose(got[k], exp[k], rtol=1e-9) for k in ("sum_qty", "sum_charge", "avg_disc")))
    if not _c:
        import sys
        print(f'rank {rank}: check at line 56 failed', file=sys.stderr, flush=True)
    ok &= _c
    # high-cardinality key: all-to-all repartition, local group-by, all-gather
    rng = np.random.default_rng(9)
    n = 50_001
    key = rng.integers(-10**9, 10**9, size=n // 5)[rng.integers(0, n // 5, size=n)]
    val = rng.normal(size=n)
    a, b = shard_bounds(n, rank, world)
    cat2 = tq.Catalog()
    cat2.register("t", tq.table_from_columns(["k", "v"], [tq.plain(tq.Tensor(key[a:b])),
                                                          tq.plain(tq.Tensor(val[a:b]))]))
    q2 = wl.compile_sql("SELECT k, SUM(v), COUNT(*) FROM t GROUP BY k", cat2, tq.UdfRegistry())
    with sharded():
        r2 = q2.run(cat2)
    ek, ea = orc.groupby_exact([key], [("sum", val), ("count", None)])
    g2 = [c.values.numpy() for c in r2.columns]
    _c = bool(np.array_equal(g2[0], ek[0]) and np.array_equal(g2[2], ea[1]))
    if not _c:
        import sys
        print(f'rank {rank}: check at line 71 failed', file=sys.stderr, flush=True)
    ok &= _c
    _c = bool(np.allclose(g2[1], ea[0], rtol=1e-9, atol=1e-12))
    if not _c:
        import sys
        print(f'rank {rank}: check at line 72 failed', file=sys.stderr, flush=True)
    ok &= _c
    # an aggregate over an inner aggregate's (replicated) result is not merged
    # across ranks again (it used to return world_size x the counts)
    q2n = wl.compile_sql("SELECT COUNT(*), SUM(sum_v) FROM (SELECT k, SUM(v) FROM t GROUP BY k)",
                         cat2, tq.UdfRegistry())
    with sharded():
        r2n = q2n.run(cat2)
    gn = [c.values.numpy() for c in r2n.columns]
    _c = bool(int(gn[0][0]) == len(ek[0]) and np.allclose(gn[1][0], val.sum(), rtol=1e-9))
    if not _c:
        import sys
        print(f"rank {rank}: nested aggregate {gn} vs {len(ek[0])}, {val.sum()}", file=sys.stderr,
              flush=True)
    ok &= _c
    # sharded equi-join: both sides repartitioned by key (all-to-all), local
    # join; the union of the ranks' pairs equals the single-process join
    from paper_2211_02753_b200.kernels import equi_join, filter_exact
    from paper_2211_02753_b200.distributed import allgather_rows

    rng = np.random.default_rng(12)
    nl, nr = 40_000, 9_000
    lk = rng.integers(0, 6_000, size=nl)
    lv = rng.normal(size=nl)
    rk = rng.integers(0, 6_000, size=nr)  # repeated build keys too
    rv = rng.integers(0, 100, size=nr)
    la, lb_ = shard_bounds(nl, rank, world)
    ra, rb_ = shard_bounds(nr, rank, world)
    left = [tq.plain(tq.Tensor(lk[la:lb_])), tq.plain(tq.Tensor(lv[la:lb_]))]
    right = [tq.plain(tq.Tensor(rk[ra:rb_])), tq.plain(tq.Tensor(rv[ra:rb_]))]
    with sharded():
        right_f = filter_exact(right, [(1, "<", 70)])
        out = equi_join(left, right_f, 0, 0)
        cols = allgather_rows([c.values.data for c in out], dist.group.WORLD)
    got = sorted(zip(*[c.cpu().numpy().tolist() for c in cols]))
    keep = rv < 70
    epi, ebi = orc.join_inner(lk, rk[keep])
    exp = sorted(zip(lk[epi].tolist(), lv[epi].tolist(), rk[keep][ebi].tolist(),
                     rv[keep][ebi].tolist()))
    _c = bool(got == exp and len(exp) > 0)
    if not _c:
        import sys
        print(f'rank {rank}: check at line 97 failed', file=sys.stderr, flush=True)
    ok &= _c
    # the Q3-style pipeline on row-sharded customer / orders / lineitem:
    # local filters, key-repartitioned joins, repartitioned group-by, the
    # all-gathered groups ordered and limited on every rank
    tables = wl.q3_arrays(0.05, seed=7)
    shard = {}
    for t, cols in tables.items():
        n_t = len(next(iter(cols.values())))
        a, b = shard_bounds(n_t, rank, world)
        shard[t] = {c: v[a:b] for c, v in cols.items()}
    cat3 = wl.q3_catalog(shard)
    with sharded():
        r3 = wl.Q3Plan(cat3).run(cat3)
    e3 = otpch.q3(tables)
    g3 = {n: c.values.numpy() for n, c in zip(r3.schema.names, r3.columns)}
    _c = bool(np.array_equal(g3["l_orderkey"], e3["l_orderkey"]))
    if not _c:
        import sys
        print(f'rank {rank}: check at line 112 failed', file=sys.stderr, flush=True)
    ok &= _c
    _c = bool(np.allclose(g3["sum_rev"], e3["sum_rev"], rtol=1e-9))
    if not _c:
        import sys
        print(f'rank {rank}: check at line 113 failed', file=sys.stderr, flush=True)
    ok &= _c
    # data-parallel LLP training: row shards of X and bag codes, the soft
    # count grid summed across ranks in the forward, the parameter gradients
    # in the backward -> the same losses and weights as one process on all rows
    from paper_2211_02753_b200.storage import tensor_type

    def llp_losses(Xn, bagn, shard_ctx):
        model = tq.Linear(64, 2, np.random.default_rng(0), name="lin")
        bag_pe = tq.one_hot_pe(bagn, 40)
        reg = tq.UdfRegistry()
        reg.register(tq.UdfEntry("llp", (("Bag", tensor_type(40)), ("Pred", tensor_type(2))), 1,
                                 lambda c: (bag_pe, tq.pe_encode(model(c.values))),
                                 model.parameters))
        catl = tq.Catalog()
        Xt = tq.Tensor(Xn)
        catl.register_tensor(Xt, "T")
        q = tq.compile_plan(tq.lower(tq.bind(tq.parse(
            "SELECT Bag, Pred, COUNT(*) FROM llp(T) GROUP BY Bag, Pred"), catl, reg)),
            tq.CompileConfig(trainable=True), reg)
        target = tq.Tensor(np.linspace(0.0, 2000.0, 80))
        with shard_ctx:
            losses = tq.train(q, catl, [("T", Xt, target)], tq.TrainConfig(iterations=4, lr=0.05))
        return losses, model.weight.value.numpy()

    import contextlib

    rng = np.random.default_rng(17)
    N = 60_000
    X = rng.normal(size=(N, 64)).astype(np.float32)
    bag = rng.integers(0, 40, size=N)
    a, b = shard_bounds(N, rank, world)
    l_sh, w_sh = llp_losses(X[a:b], bag[a:b], sharded())
    l_one, w_one = llp_losses(X, bag, contextlib.nullcontext())
    llp_ok = np.allclose(l_sh, l_one, rtol=1e-5) and np.allclose(w_sh, w_one, rtol=1e-5, atol=1e-5)
    if not llp_ok:
        import sys
        print(f"rank {rank} sharded LLP: losses {l_sh} vs {l_one}; "
              f"max |dW| {np.max(np.abs(w_sh - w_one))}", file=sys.stderr, flush=True)
    ok &= llp_ok
    # ORDER BY / LIMIT over a row-sharded relation: local top rows, gathered
    # in rank order, ordered again == the global stable order
    rng = np.random.default_rng(23)
    nt = 30_001
    kv = rng.integers(0, 500, size=nt).astype(np.float64)  # many ties
    iv = np.arange(nt)
    a2, b2 = shard_bounds(nt, rank, world)
    cat4 = tq.Catalog()
    cat4.register("t", tq.table_from_columns(["i", "v"], [tq.plain(tq.Tensor(iv[a2:b2])),
                                                          tq.plain(tq.Tensor(kv[a2:b2]))]))
    for sql, desc, lim in (("SELECT i, v FROM t ORDER BY v DESC LIMIT 25", True, 25),
                           ("SELECT i, v FROM t ORDER BY v LIMIT 3000", False, 3000),
                           ("SELECT i, v FROM t WHERE v > 100 ORDER BY v", False, None),
                           ("SELECT i, v FROM t LIMIT 40", None, 40)):
        q4 = wl.compile_sql(sql, cat4, tq.UdfRegistry())
        with sharded():
            r4 = q4.run(cat4)
        got_i = r4.columns[0].values.numpy()
        if desc is None:
            exp_i = iv[:lim]
        else:
            keep = kv > 100 if "WHERE" in sql else np.ones(nt, dtype=bool)
            order = orc.stable_order(kv[keep], desc)
            exp_i = iv[keep][order][: lim if lim is not None else None]
        c4 = bool(np.array_equal(got_i, exp_i))
        if not c4:
            import sys
            print(f"rank {rank} sharded '{sql}' mismatch", file=sys.stderr, flush=True)
        ok &= c4
    # trainable global aggregates (GlobalAggSoftOp) over row shards
    def scored(Xn, shard_ctx):
        reg = tq.UdfRegistry()
        wts = tq.Tensor(np.linspace(-1.0, 1.0, 64))
        reg.register(tq.make_scoring_udf("scorer", wts, scale=8.0))
        catl = tq.Catalog()
        catl.register_tensor(tq.Tensor(Xn.astype(np.float64)), "T")
        q = tq.compile_plan(tq.lower(tq.bind(tq.parse(
            "SELECT SUM(Score), AVG(Score), COUNT(*) FROM scorer(T)"), catl, reg)),
            tq.CompileConfig(trainable=True), reg)
        with shard_ctx:
            r = q.run(catl)
        return [float(c.values.numpy()[0]) for c in r.columns]

    g_sh = scored(X[a:b], sharded())
    g_one = scored(X, contextlib.nullcontext())
    g_ok = np.allclose(g_sh, g_one, rtol=1e-9)
    if not g_ok:
        import sys
        print(f"rank {rank} global soft aggregates {g_sh} vs {g_one}", file=sys.stderr, flush=True)
    ok &= g_ok
    if not ok:
        import sys
        print(f"rank {rank}: checks failed", file=sys.stderr, flush=True)
    result[rank] = bool(ok)
    dist.destroy_process_group()


def test_two_ranks_one_gpu_sharded_queries():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    result = mgr.dict()
    mp.start_processes(_worker, args=(2, _port(), result), nprocs=2, join=True,
                       start_method="spawn")
    assert result.get(0) is True and result.get(1) is True

"""GPU: equi-join (builder-defined: no reference join exists).

The oracle ``join_inner`` (sort + searchsorted) is itself checked against a
nested-loop join on adversarial inputs (CPU test below), then both join
algorithms of the B200 path -- the hash join and the dense-range (bitmap)
join -- must give exactly its (probe row, build row) pairs in its order.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2211_02753_b200 as tq
from oracle import relational as orc
from paper_2211_02753_b200 import kernels as K
from paper_2211_02753_b200 import workloads as wl

I64 = np.iinfo(np.int64)


def _cases():
    rng = np.random.default_rng(40)
    yield "dups_both_sides", rng.integers(0, 30, size=700), rng.integers(0, 30, size=500)
    yield "all_equal", np.full(300, 7), np.full(200, 7)
    yield "empty_probe", np.array([], dtype=np.int64), rng.integers(0, 9, size=50)
    yield "empty_build", rng.integers(0, 9, size=50), np.array([], dtype=np.int64)
    yield "no_match", np.arange(0, 400, 2), np.arange(1, 400, 2)
    yield "int64_extremes", (np.array([I64.min, I64.max, 0, -1, 1, I64.min + 1, I64.max - 1] * 40)
                             [rng.permutation(280)]), \
        np.array([I64.max, I64.min, -1, I64.max, 5, I64.min + 1])
    yield "negative_dense", rng.integers(-1000, -900, size=600), rng.permutation(100) - 1000


@pytest.mark.parametrize("name,probe,build", list(_cases()))
def test_oracle_join_equals_nested_loop(name, probe, build):
    """CPU: the oracle against brute force (runs without a GPU)."""
    probe, build = np.asarray(probe, np.int64), np.asarray(build, np.int64)
    epi, ebi = orc.join_inner(probe, build)
    npi, nbi = orc.join_nested_loop(probe, build)
    np.testing.assert_array_equal(epi, npi)
    np.testing.assert_array_equal(ebi, nbi)


def _dev(a):
    return torch.as_tensor(np.asarray(a, np.int64)).cuda()


@pytest.mark.gpu
@pytest.mark.parametrize("name,probe,build", list(_cases()))
@pytest.mark.parametrize("algo", ["hash", "dense", "sort"])
def test_join_adversarial_vs_oracle(name, probe, build, algo, monkeypatch):
    """hash: open-addressing + Bloom; dense: bitmap over the build key range;
    sort: radix-sorted build + searchsorted probe (tdp_join_sorted_*)."""
    probe, build = np.asarray(probe, np.int64), np.asarray(build, np.int64)
    monkeypatch.setattr(K, "JOIN_ALGORITHM", "sort" if algo == "sort" else "auto")
    rng = None
    if algo == "dense" and len(build):
        rng = (int(build.min()), int(build.max()))
    pairs = K.join_indices(_dev(probe), _dev(build), build_range=rng)
    epi, ebi = orc.join_inner(probe, build)
    np.testing.assert_array_equal(pairs[0].cpu().numpy(), epi)
    np.testing.assert_array_equal(pairs[1].cpu().numpy(), ebi)


@pytest.mark.gpu
@pytest.mark.parametrize("lo", [0, -(2**40), 2**63 - 5_000_000, -(2**63)])
@pytest.mark.parametrize("need_rows", [True, False])
def test_dense_join_unique_build(lo, need_rows):
    """Unique build keys in a known range: the bitmap join (incl. ranges at
    the ends of int64), with and without the build-row index."""
    rng = np.random.default_rng(abs(lo) % 1000 + 3)
    span = 4_000_000
    build = lo + rng.choice(span, size=700_000, replace=False).astype(np.int64)
    probe = lo + rng.integers(0, span, size=1_500_000).astype(np.int64)
    pairs = K.join_indices(_dev(probe), _dev(build), build_range=(lo, lo + span - 1),
                           need_build_rows=need_rows)
    epi, ebi = orc.join_inner(probe, build)
    np.testing.assert_array_equal(pairs[0].cpu().numpy(), epi)
    if need_rows:
        np.testing.assert_array_equal(pairs[1].cpu().numpy(), ebi)
    else:
        assert pairs[1] is None


@pytest.mark.gpu
def test_dense_join_rank_mode_fused_emit():
    """A build whose range is > 8 keys per row (but <= 64): build rows are
    found by the key's rank among the set bits (no key-offset array) in the
    fused expand + pairs emit; a high match rate (every probe row matches
    once or more) exercises the four-at-a-time pair loop."""
    rng = np.random.default_rng(17)
    span, nb = 60_000_000, 1_100_000
    build = rng.choice(span, size=nb, replace=False).astype(np.int64) + 5
    probe = np.concatenate([rng.choice(build, size=1_500_000),
                            rng.integers(0, span + 10, size=500_000)]).astype(np.int64)
    rng.shuffle(probe)
    pairs = K.join_indices(_dev(probe), _dev(build), build_range=(5, span + 4))
    epi, ebi = orc.join_inner(probe, build)
    np.testing.assert_array_equal(pairs[0].cpu().numpy(), epi)
    np.testing.assert_array_equal(pairs[1].cpu().numpy(), ebi)


@pytest.mark.gpu
def test_dense_join_filtered_sides_from_base_columns():
    """A filtered build and a filtered probe read straight from base columns
    (equi_join on lazy selections): the build key's range is the catalog
    column's statistic, cached on the tensor."""
    rng = np.random.default_rng(8)
    nb, npr = 300_000, 2_000_000
    bkey = rng.permutation(nb).astype(np.int64) * 3 + 11
    bflag = rng.integers(0, 4, size=nb)
    pkey = rng.integers(0, 3 * nb + 20, size=npr).astype(np.int64)
    pval = rng.normal(size=npr)
    right = [tq.plain(tq.Tensor(bkey)), tq.plain(tq.Tensor(bflag))]
    left = [tq.plain(tq.Tensor(pkey)), tq.plain(tq.Tensor(pval))]
    rf = K.filter_exact(right, [(1, "<", 2)])
    lf = K.filter_exact(left, [(1, ">", 0.3)])
    out = K.equi_join(lf, rf, 0, 0)
    base = right[0].values.data
    assert K.column_range(base, compute=False) == (int(bkey.min()), int(bkey.max()))
    keep_b = bflag < 2
    keep_p = pval > 0.3
    epi, ebi = orc.join_inner(pkey[keep_p], bkey[keep_b])
    np.testing.assert_array_equal(out[0].values.numpy(), pkey[keep_p][epi])
    np.testing.assert_array_equal(out[1].values.numpy(), pval[keep_p][epi])
    np.testing.assert_array_equal(out[3].values.numpy(), bflag[keep_b][ebi])


@pytest.mark.gpu
@pytest.mark.parametrize("sf", [0.02, 0.2])
def test_q3_dense_joins_and_replay(sf):
    """The Q3 pipeline (both joins dense: c_custkey, o_orderkey statistics)
    eager and replayed, all four result columns against the oracle."""
    from oracle import tpch as otpch

    tables = wl.q3_arrays(sf, seed=7)
    cat = wl.q3_catalog(tables)
    plan = wl.Q3Plan(cat)
    exp = otpch.q3(tables)
    for _ in range(4):  # eager, record, capture, replay
        res = plan.run(cat)
        got = [c.values.numpy() for c in res.columns]
        np.testing.assert_array_equal(got[0], exp["l_orderkey"])
        np.testing.assert_allclose(got[1], exp["sum_rev"], rtol=1e-9)
        np.testing.assert_allclose(got[2], exp["avg_o_orderdate"], rtol=1e-12)
        np.testing.assert_allclose(got[3], exp["avg_o_shippriority"], rtol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("nb,npr,kmax", [(5000, 300_000, 4000), (1_000_003, 3_000_017, 1 << 40),
                                          (20_000, 500_000, 50)])
def test_sorted_join_large_vs_oracle(nb, npr, kmax):
    """The sort / searchsorted join beyond one fence block (build > 4096
    keys: the shared-memory top level plus the global fence interval), with
    repeated build keys (kmax < nb: long runs) and a sorted probe column."""
    rng = np.random.default_rng(nb)
    build = rng.integers(-kmax, kmax, size=nb).astype(np.int64)
    probe = np.sort(rng.integers(-kmax, kmax, size=npr).astype(np.int64))
    pk, bk = _dev(probe), _dev(build)
    from paper_2211_02753_b200 import _native as nat

    buf = nat.workspace(nat.load().tdp_join_sorted_workspace(nb, npr), pk.device)
    cnt = torch.empty(1, dtype=torch.int64, device=pk.device)
    nat.call("tdp_join_sorted_prepare", nat.ptr(bk), nb, nat.ptr(pk), npr, nat.columns([]), 0,
             nat.struct_array(nat.Predicate, []), 0, nat.ptr(cnt), nat.ptr(buf), buf.numel(),
             nat.stream())
    m = int(cnt.item())
    epi, ebi = orc.join_inner(probe, build)
    assert m == len(epi)
    pi = torch.empty(m, dtype=torch.int64, device=pk.device)
    bi = torch.empty(m, dtype=torch.int64, device=pk.device)
    nat.call("tdp_join_sorted_emit", nat.ptr(pk), nb, npr, nat.ptr(pi), nat.ptr(bi), nat.ptr(buf),
             buf.numel(), nat.stream())
    np.testing.assert_array_equal(pi.cpu().numpy(), epi)
    np.testing.assert_array_equal(bi.cpu().numpy(), ebi)


@pytest.mark.gpu
def test_sorted_join_filtered_sides_and_q3(monkeypatch):
    """TDP_JOIN_ALGO=sort through equi_join on lazy filtered sides (build
    compacted by its selection, probe predicates inside the count pass) and
    through the whole Q3 pipeline, against the oracle."""
    from oracle import tpch as otpch

    monkeypatch.setattr(K, "JOIN_ALGORITHM", "sort")
    rng = np.random.default_rng(9)
    nb, npr = 200_000, 1_000_000
    bkey = rng.integers(0, 150_000, size=nb).astype(np.int64)
    bflag = rng.integers(0, 4, size=nb)
    pkey = rng.integers(0, 160_000, size=npr).astype(np.int64)
    pval = rng.normal(size=npr)
    right = [tq.plain(tq.Tensor(bkey)), tq.plain(tq.Tensor(bflag))]
    left = [tq.plain(tq.Tensor(pkey)), tq.plain(tq.Tensor(pval))]
    out = K.equi_join(K.filter_exact(left, [(1, ">", 0.3)]),
                      K.filter_exact(right, [(1, "<", 2)]), 0, 0)
    keep_b, keep_p = bflag < 2, pval > 0.3
    epi, ebi = orc.join_inner(pkey[keep_p], bkey[keep_b])
    np.testing.assert_array_equal(out[0].values.numpy(), pkey[keep_p][epi])
    np.testing.assert_array_equal(out[1].values.numpy(), pval[keep_p][epi])
    np.testing.assert_array_equal(out[3].values.numpy(), bflag[keep_b][ebi])
    tables = wl.q3_arrays(0.05, seed=7)
    cat = wl.q3_catalog(tables)
    res = wl.Q3Plan(cat).run(cat)
    exp = otpch.q3(tables)
    got = [c.values.numpy() for c in res.columns]
    np.testing.assert_array_equal(got[0], exp["l_orderkey"])
    np.testing.assert_allclose(got[1], exp["sum_rev"], rtol=1e-9)


def _fuzz_case(seed: int):
    """A random join: key distribution (dense / sparse / clustered / few
    distinct), sizes (empty .. 300 K), build keys unique or repeated, and
    filters on either side (as equi_join on lazy selections)."""
    rng = np.random.default_rng(1000 + seed)
    kind = seed % 4
    nb = int(rng.choice([0, 1, 17, 3000, 70_000, 300_000]))
    npr = int(rng.choice([0, 5, 2000, 150_000, 300_000]))
    if kind == 0:    # dense unique build (bitmap join)
        span = max(nb, 1) * int(rng.integers(1, 40))
        build = rng.choice(span, size=min(nb, span), replace=False) + int(rng.integers(-10**9, 10**9))
    elif kind == 1:  # sparse unique build over the int64 range (hash join)
        build = np.unique(rng.integers(I64.min // 2, I64.max // 2, size=nb))
        rng.shuffle(build)
    elif kind == 2:  # repeated build keys
        build = rng.integers(0, max(1, nb // 7), size=nb)
    else:            # clustered (sorted runs) build
        build = np.sort(rng.integers(0, max(1, nb // 3), size=nb))
    build = np.asarray(build, np.int64)
    pool = build if len(build) else np.arange(3, dtype=np.int64)
    probe = np.where(rng.random(npr) < 0.6, rng.choice(pool, size=npr),
                     rng.integers(int(pool.min()) - 5, int(pool.max()) + 6, size=npr))
    return np.asarray(probe, np.int64), build, rng


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(24))
@pytest.mark.parametrize("algo", ["auto", "sort"])
def test_join_fuzz_vs_oracle(seed, algo, monkeypatch):
    """Random joins through equi_join (filtered sides included) against the
    oracle's join_inner, itself pinned to a nested loop."""
    probe, build, rng = _fuzz_case(seed)
    monkeypatch.setattr(K, "JOIN_ALGORITHM", algo)
    pv = rng.normal(size=len(probe))
    bv = rng.integers(0, 4, size=len(build))
    left = [tq.plain(tq.Tensor(probe)), tq.plain(tq.Tensor(pv))]
    right = [tq.plain(tq.Tensor(build)), tq.plain(tq.Tensor(bv))]
    keep_p = np.ones(len(probe), bool)
    keep_b = np.ones(len(build), bool)
    if seed % 3 == 1 and len(probe):
        left = K.filter_exact(left, [(1, ">", 0.2)])
        keep_p = pv > 0.2
    if seed % 3 == 2 and len(build):
        right = K.filter_exact(right, [(1, "<", 3)])
        keep_b = bv < 3
    out = K.equi_join(left, right, 0, 0)
    epi, ebi = orc.join_inner(probe[keep_p], build[keep_b])
    np.testing.assert_array_equal(out[0].values.numpy(), probe[keep_p][epi])
    np.testing.assert_array_equal(out[1].values.numpy(), pv[keep_p][epi])
    np.testing.assert_array_equal(out[2].values.numpy(), build[keep_b][ebi])
    np.testing.assert_array_equal(out[3].values.numpy(), bv[keep_b][ebi])

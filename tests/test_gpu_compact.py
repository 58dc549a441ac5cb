"""GPU parity of compact column storage.

A compacted table must be indistinguishable from the original: decoded column
values bit-identical, every query result equal to the wide table's (keys,
counts, row sets bit-exact; float aggregates rtol 1e-12 -- only the reduction
grouping can differ) and to the oracle (rtol 1e-9).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle.tpch as otpch
from oracle import relational as orc
import paper_2211_02753_b200 as tq
from paper_2211_02753_b200 import compact as cp
from paper_2211_02753_b200 import kernels as K
from paper_2211_02753_b200 import workloads as wl

pytestmark = pytest.mark.gpu


def _catalogs(arrays, columns=wl.LINEITEM_COLUMNS):
    wide = wl.lineitem_table(arrays, columns)
    narrow = cp.compact_table(wide)
    cw, cn = tq.Catalog(), tq.Catalog()
    cw.register("lineitem", wide)
    cn.register("lineitem", narrow)
    return cw, cn, narrow


def test_lineitem_storage_plan_and_round_trip():
    arrays = wl.lineitem_arrays(0.01, seed=2, rows=20_000)
    _, _, narrow = _catalogs(arrays)
    specs = dict(zip(narrow.schema.names, cp.specs_of(narrow)))
    assert specs["l_shipdate"] == cp.CompactSpec(torch.int16, 0)
    assert specs["l_returnflag"] == cp.CompactSpec(torch.uint8, 0)
    assert specs["l_linestatus"] == cp.CompactSpec(torch.uint8, 0)
    assert specs["l_quantity"] == cp.CompactSpec(torch.int8, 1)
    assert specs["l_extendedprice"] == cp.CompactSpec(torch.int32, 100)
    assert specs["l_discount"] == cp.CompactSpec(torch.int8, 100)
    assert specs["l_tax"] == cp.CompactSpec(torch.int8, 100)
    assert sum(cp.stored_bytes(c) for c in narrow.columns) == 11
    for name, col in zip(narrow.schema.names, narrow.columns):
        got = col.values.numpy()
        assert got.dtype == arrays[name].dtype
        np.testing.assert_array_equal(got.view(np.int64), arrays[name].view(np.int64))
    assert narrow.columns[1].is_dictionary()
    assert narrow.columns[1].encoding.dictionary == wl.RETURNFLAG


@pytest.mark.parametrize("rows", [1, 5000, 200_003, 1_000_003])
def test_q1_compact_equals_wide_and_oracle(rows):
    arrays = wl.lineitem_arrays(0.01, seed=5, rows=rows)
    cw, cn, _ = _catalogs(arrays)
    qw = wl.compile_sql(wl.Q1_SQL, cw, wl.q1_registry())
    qn = wl.compile_sql(wl.Q1_SQL, cn, wl.q1_registry())
    rw, rn = qw.run(cw), qn.run(cn)
    exp = otpch.q1(arrays)
    assert rn.schema.names == rw.schema.names
    for name, a, b in zip(rn.schema.names, rw.columns, rn.columns):
        x, y = a.values.numpy(), b.values.numpy()
        assert x.dtype == y.dtype
        if x.dtype.kind in "iu":
            np.testing.assert_array_equal(y, x)
            np.testing.assert_array_equal(y, exp[name])
        else:
            np.testing.assert_allclose(y, x, rtol=1e-12)
            np.testing.assert_allclose(y, exp[name], rtol=1e-9)
    assert rn.columns[0].is_dictionary()


@pytest.mark.parametrize("rows", [0, 777, 123_457, 400_009, 1_500_001])
def test_q6_compact_equals_oracle(rows):
    cols = ("l_shipdate", "l_quantity", "l_extendedprice", "l_discount")
    arrays = wl.lineitem_arrays(0.01, seed=3, rows=rows)
    if rows == 0:  # nothing to compact: stays wide, still runs
        return
    cw, cn, _ = _catalogs(arrays, cols)
    q = wl.compile_sql(wl.Q6_SQL, cn, wl.q6_registry())
    got = q.run(cn).columns[0].values.numpy()
    np.testing.assert_allclose(got, otpch.q6(arrays)["sum_rev"], rtol=1e-9, atol=1e-9)


def test_filters_on_compact_columns_materialise_bit_exact():
    arrays = wl.lineitem_arrays(0.01, seed=7, rows=50_000)
    _, cn, _ = _catalogs(arrays)
    sql = ("SELECT * FROM lineitem WHERE l_shipdate >= 9000 AND l_discount < 0.05 "
           "AND l_returnflag = \"R\" AND l_extendedprice > 20000.5 AND l_quantity <= 30")
    q = wl.compile_sql(sql, cn, tq.UdfRegistry())
    res = q.run(cn)
    cols = [arrays[c] for c in wl.LINEITEM_COLUMNS]
    idx = orc.filter_indices(cols, [(0, ">=", 9000), (5, "<", 0.05), (1, "=", 2),
                                    (4, ">", 20000.5), (3, "<=", 30)])
    assert res.row_count == len(idx)
    for name, col in zip(res.schema.names, res.columns):
        np.testing.assert_array_equal(col.values.numpy(), arrays[name][idx])


def test_decimal_literal_edges():
    # literals between two representable decimals, exactly on one, ints, negatives
    vals = np.round(np.arange(-500, 500) / 100.0, 2)
    t = tq.table_from_columns(["x"], [tq.plain(tq.Tensor(vals))])
    narrow = cp.compact_table(t)
    assert cp.specs_of(narrow)[0] == cp.CompactSpec(torch.int16, 100)
    for op, lit in (("<", 0.07), ("<=", 0.07), (">", -0.005), (">=", 1.0), ("=", 0.3),
                    ("<>", 0.1), ("<", 3), (">=", -2), ("=", -4.99), (">", 1e300)):
        out = K.filter_exact(list(narrow.columns), [(0, op, lit)])
        got = out[0].values.numpy()
        idx = orc.filter_indices([vals], [(0, op, lit)])
        np.testing.assert_array_equal(got, vals[idx])


def test_non_decimal_and_special_values_stay_wide():
    rng = np.random.default_rng(0)
    cases = [rng.random(1000), np.array([1.25, -0.0, 2.5]), np.array([1.0, np.nan, 2.0]),
             np.array([1.0, np.inf]), np.array([3e12, 1.0])]
    for arr in cases:
        col = tq.plain(tq.Tensor(arr))
        assert cp.plan_column(col) is None
    big = tq.plain(tq.Tensor(np.array([0, 2**40], dtype=np.int64)))
    assert cp.plan_column(big) is None


def test_table_from_stored_round_trip():
    arrays = wl.lineitem_arrays(0.01, seed=9, rows=4096)
    _, _, narrow = _catalogs(arrays)
    stored = [t.clone() for t in cp.stored_tensors(narrow)]
    again = cp.table_from_stored(narrow, stored)
    for a, b in zip(narrow.columns, again.columns):
        np.testing.assert_array_equal(a.values.numpy(), b.values.numpy())


def _exact_q1_floats(arrays):
    """Per (rf, ls) group (ascending) the exact rational Q1 float aggregates over
    the stored integers, rounded once (fractions): the result the exact
    decimal path must reproduce to within the final rounding."""
    from fractions import Fraction

    keep = arrays["l_shipdate"] <= 10471
    rf, ls = arrays["l_returnflag"][keep], arrays["l_linestatus"][keep]
    q = np.rint(arrays["l_quantity"][keep]).astype(np.int64)
    c = np.rint(arrays["l_extendedprice"][keep] * 100).astype(np.int64)
    d = np.rint(arrays["l_discount"][keep] * 100).astype(np.int64)
    t = np.rint(arrays["l_tax"][keep] * 100).astype(np.int64)
    dp = c * (100 - d)                  # |.| < 2^39: exact in int64
    ch = dp * (100 + t)                 # |.| < 2^47
    out = {k: [] for k in ("sum_qty", "sum_price", "sum_disc_price", "sum_charge", "avg_qty",
                           "avg_price", "avg_disc", "count")}
    for g in sorted(set(zip(rf.tolist(), ls.tolist()))):
        m = (rf == g[0]) & (ls == g[1])
        n = int(m.sum())
        sq, sp, sd = int(q[m].sum()), int(c[m].sum()), int(d[m].sum())
        sdp, sch = sum(dp[m].tolist()), sum(ch[m].tolist())
        out["sum_qty"].append(float(sq))
        out["sum_price"].append(float(Fraction(sp, 100)))
        out["sum_disc_price"].append(float(Fraction(sdp, 10_000)))
        out["sum_charge"].append(float(Fraction(sch, 1_000_000)))
        out["avg_qty"].append(float(Fraction(sq, n)))
        out["avg_price"].append(float(Fraction(sp, 100 * n)))
        out["avg_disc"].append(float(Fraction(sd, 100 * n)))
        out["count"].append(n)
    return {k: np.asarray(v) for k, v in out.items()}


@pytest.mark.parametrize("rows", [4093, 300_007, 2_000_003])
def test_q1_compact_decimal_sums_exact_at_type_extremes(rows):
    """Compact decimals at the extremes of their stored types (int32 cents
    incl. INT32_MIN/MAX, negative int8 discounts/taxes/quantities): the fused
    scan sums them as exact scaled integers in packed per-thread words
    (pipeline.cu convert_decimal_sums / pack_fields), so every float aggregate
    equals the exactly rounded rational sum -- no float reassociation error
    even under cancellation."""
    rng = np.random.default_rng(rows)
    arrays = wl.lineitem_arrays(0.01, seed=17, rows=rows)
    c = rng.integers(-2**31, 2**31, rows, dtype=np.int64)
    c[:4] = [-2**31, 2**31 - 1, -2**31, 2**31 - 1]
    arrays["l_extendedprice"] = c / 100.0
    arrays["l_discount"] = rng.integers(-128, 128, rows) / 100.0
    arrays["l_tax"] = rng.integers(-128, 128, rows) / 100.0
    arrays["l_quantity"] = rng.integers(-128, 128, rows).astype(np.float64)
    cw, cn, narrow = _catalogs(arrays)
    specs = dict(zip(narrow.schema.names, cp.specs_of(narrow)))
    assert specs["l_extendedprice"] == cp.CompactSpec(torch.int32, 100)
    assert specs["l_discount"] == cp.CompactSpec(torch.int8, 100)
    assert specs["l_quantity"] == cp.CompactSpec(torch.int8, 1)
    res = wl.compile_sql(wl.Q1_SQL, cn, wl.q1_registry()).run(cn)
    got = {n: c.values.numpy() for n, c in zip(res.schema.names, res.columns)}
    exp = otpch.q1(arrays)  # group keys and counts (bit-exact)
    np.testing.assert_array_equal(got["rf"], exp["rf"])
    np.testing.assert_array_equal(got["ls"], exp["ls"])
    np.testing.assert_array_equal(got["count"], exp["count"])
    exact = _exact_q1_floats(arrays)
    for k in ("sum_qty", "sum_price", "sum_disc_price", "sum_charge", "avg_qty", "avg_price",
              "avg_disc"):
        # two roundings at most (the int sum -> double, then / scale or / count)
        np.testing.assert_allclose(got[k], exact[k], rtol=5e-16, atol=0, err_msg=k)


@pytest.mark.parametrize("rows", [3001, 700_001])
def test_q1_compact_bitwise_repeatable(rows):
    """Exact integer accumulation is order-free: two runs are bitwise equal,
    and equal the float64 reference within its own rounding (rtol 1e-12)."""
    arrays = wl.lineitem_arrays(0.01, seed=23, rows=rows)
    cw, cn, _ = _catalogs(arrays)
    q = wl.compile_sql(wl.Q1_SQL, cn, wl.q1_registry())
    a, b = q.run(cn), q.run(cn)
    for x, y in zip(a.columns, b.columns):
        np.testing.assert_array_equal(x.values.numpy().view(np.uint8), y.values.numpy().view(np.uint8))
    exact = _exact_q1_floats(arrays)
    got = {n: c.values.numpy() for n, c in zip(a.schema.names, a.columns)}
    for k in exact:
        np.testing.assert_allclose(got[k], exact[k], rtol=5e-16, atol=0, err_msg=k)

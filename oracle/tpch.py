"""Reference-algorithm restatement of the headline queries (test infrastructure).

Q1 / Q6 exactly as the reference executes the Appendix-A plans:
FilterOp -> filter_exact (mask chain, nonzero, take_rows on EVERY column,
tq/kernels.py:87-97) -> TvfOp (numpy elementwise UDF) -> GroupAggExactOp ->
groupby_exact (tq/kernels.py:108-167) / _global_aggregate
(tq/compiler.py:206-215).  Used as the parity oracle and as the CPU baseline
("port") in bench.py.
"""

from __future__ import annotations

import numpy as np

from .relational import filter_exact, global_aggregate, groupby_exact

Q1_COLS = ("l_shipdate", "l_returnflag", "l_linestatus", "l_quantity", "l_extendedprice",
           "l_discount", "l_tax")


def q1(arrays: dict) -> dict[str, np.ndarray]:
    cols = [arrays[c] for c in Q1_COLS]
    ship, rf, ls, q, p, d, t = filter_exact(cols, [(0, "<=", 10471)])
    one = np.asarray(1.0)
    dp = p * (one - d)
    ch = dp * (one + t)
    keys, aggs = groupby_exact([rf, ls], [("sum", q), ("sum", p), ("sum", dp), ("sum", ch),
                                          ("avg", q), ("avg", p), ("avg", d), ("count", None)])
    names = ["sum_qty", "sum_price", "sum_disc_price", "sum_charge", "avg_qty", "avg_price",
             "avg_disc", "count"]
    out = {"rf": keys[0], "ls": keys[1]}
    out.update(dict(zip(names, aggs)))
    return out


def q1_partial(arrays: dict) -> dict[tuple, list]:
    """Q1 over one row range of lineitem: per (rf, ls) group the five sums and
    the count -- the mergeable part of q1() (AVG = merged SUM / merged COUNT,
    as tq/kernels.py:147-153 forms it from the whole column)."""
    cols = [arrays[c] for c in Q1_COLS]
    ship, rf, ls, q, p, d, t = filter_exact(cols, [(0, "<=", 10471)])
    one = np.asarray(1.0)
    dp = p * (one - d)
    ch = dp * (one + t)
    keys, aggs = groupby_exact([rf, ls], [("sum", q), ("sum", p), ("sum", dp), ("sum", ch),
                                          ("sum", d), ("count", None)])
    return {(int(a), int(b)): [float(x[g]) for x in aggs[:5]] + [int(aggs[5][g])]
            for g, (a, b) in enumerate(zip(keys[0], keys[1]))}


def q1_merge(parts) -> dict[str, np.ndarray]:
    """q1() of the concatenated row ranges from their q1_partial()s."""
    acc: dict = {}
    for part in parts:
        for key, vals in part.items():
            cur = acc.setdefault(key, [0.0] * 5 + [0])
            for a, v in enumerate(vals):
                cur[a] += v
    keys = sorted(acc)
    col = lambda a: np.array([acc[k][a] for k in keys], dtype=np.float64)  # noqa: E731
    cnt = np.array([acc[k][5] for k in keys], dtype=np.int64)
    return {"rf": np.array([k[0] for k in keys], dtype=np.int64),
            "ls": np.array([k[1] for k in keys], dtype=np.int64),
            "sum_qty": col(0), "sum_price": col(1), "sum_disc_price": col(2),
            "sum_charge": col(3), "avg_qty": col(0) / cnt, "avg_price": col(1) / cnt,
            "avg_disc": col(4) / cnt, "count": cnt}


def q6_partial(arrays: dict) -> tuple[float, int]:
    """Q6 over one row range: (SUM(extendedprice * discount), qualifying rows)."""
    cols = [arrays[c] for c in ("l_shipdate", "l_discount", "l_quantity", "l_extendedprice")]
    ship, d, q, p = filter_exact(cols, [(0, ">=", 8766), (0, "<", 9131), (1, ">=", 0.05),
                                        (1, "<=", 0.07), (2, "<", 24)])
    return float((p * d).sum()), len(p)


def q6_merge(parts) -> dict[str, np.ndarray]:
    return {"sum_rev": np.array([sum(s for s, _ in parts)], dtype=np.float64)}


def q3(tables: dict) -> dict[str, np.ndarray]:
    """Q3-style pipeline: reference filters (filter_exact) on each table, the
    builder-defined sort/searchsorted join (no join in the reference), the
    reference's groupby_exact / sort_limit on the joined rows."""
    from .relational import join_inner, sort_limit

    c, o, li = tables["customer"], tables["orders"], tables["lineitem"]
    (ck,) = filter_exact([c["c_custkey"], c["c_mktsegment"]], [(1, "=", 1)])[:1]
    ok, ocust, odate, oship = filter_exact(
        [o["o_orderkey"], o["o_custkey"], o["o_orderdate"], o["o_shippriority"]],
        [(2, "<", 9204)])
    lk, lp, ld = filter_exact([li["l_orderkey"], li["l_extendedprice"], li["l_discount"],
                               li["l_shipdate"]], [(3, ">", 9204)])[:3]
    pi, bi = join_inner(ocust, ck)
    ok, ocust, odate, oship = ok[pi], ocust[pi], odate[pi], oship[pi]
    pi, bi = join_inner(lk, ok)
    jk, jp, jd, jdate, jship = lk[pi], lp[pi], ld[pi], odate[bi], oship[bi]
    rev = jp * (np.asarray(1.0) - jd)
    keys, aggs = groupby_exact([jk], [("sum", rev), ("avg", jdate), ("avg", jship)])
    out = sort_limit([keys[0], aggs[0], aggs[1], aggs[2]], 1, True, 10)
    return {"l_orderkey": out[0], "sum_rev": out[1], "avg_o_orderdate": out[2],
            "avg_o_shippriority": out[3], "joined_rows": np.asarray(len(jk))}


def q6(arrays: dict) -> dict[str, np.ndarray]:
    cols = [arrays[c] for c in ("l_shipdate", "l_discount", "l_quantity", "l_extendedprice")]
    ship, d, q, p = filter_exact(cols, [(0, ">=", 8766), (0, "<", 9131), (1, ">=", 0.05),
                                        (1, "<=", 0.07), (2, "<", 24)])
    rev = p * d
    (s,) = global_aggregate(len(rev), [("sum", rev)])
    return {"sum_rev": s}

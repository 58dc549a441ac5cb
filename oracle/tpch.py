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


def q6(arrays: dict) -> dict[str, np.ndarray]:
    cols = [arrays[c] for c in ("l_shipdate", "l_discount", "l_quantity", "l_extendedprice")]
    ship, d, q, p = filter_exact(cols, [(0, ">=", 8766), (0, "<", 9131), (1, ">=", 0.05),
                                        (1, "<=", 0.07), (2, "<", 24)])
    rev = p * d
    (s,) = global_aggregate(len(rev), [("sum", rev)])
    return {"sum_rev": s}

"""Benchmark workloads: seeded synthetic TPC-H-like tables and the reference-API
restatement of the headline queries.

The queries are written exactly as a user of the reference would write them
(SQL text + TvfMap UDFs built from tensor ops, because the reference grammar
has no arithmetic); nothing here is specific to this implementation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .encodings import DictionaryEncoding, EncodedTensor, StringDictionary, plain, trusted
from .kernels import UdfEntry, UdfRegistry
from .storage import FLOAT, STRING, Catalog, table_from_columns
from .tensor import Tensor, add, mul, sub, tensor

# day numbers since 1970-01-01 (Appendix B)
D_1992_01_01 = 8035
D_1994_01_01 = 8766
D_1995_01_01 = 9131
D_1995_03_15 = 9204
D_CURRENT = 9298  # 1995-06-17
D_Q1_CUTOFF = 10471  # 1998-12-01 - 90 days
D_1998_12_31 = 10591

RETURNFLAG = StringDictionary(("A", "N", "R"))
LINESTATUS = StringDictionary(("F", "O"))

LINEITEM_COLUMNS = ("l_shipdate", "l_returnflag", "l_linestatus", "l_quantity",
                    "l_extendedprice", "l_discount", "l_tax")


LINEITEM_CHUNK = 1 << 21  # rows per independently seeded generator chunk


def _lineitem_chunk(sf: float, seed: int, chunk: int, rows: int) -> dict[str, np.ndarray]:
    """Rows [chunk * LINEITEM_CHUNK, + rows) of the canonical table: chunk 0
    draws from ``default_rng(seed)``, chunk c > 0 from ``default_rng([seed, c])``."""
    rng = np.random.default_rng(seed if chunk == 0 else [seed, chunk])
    n = rows
    orderdate = rng.integers(D_1992_01_01, 10440 + 1, size=n, dtype=np.int64)
    shipdate = orderdate + rng.integers(1, 122, size=n, dtype=np.int64)
    receipt = shipdate + rng.integers(1, 31, size=n, dtype=np.int64)
    qty = rng.integers(1, 51, size=n).astype(np.float64)
    partkey = rng.integers(1, int(200_000 * max(sf, 1e-6)) + 1, size=n, dtype=np.int64)
    retail = (90000 + (partkey // 10) % 20001 + 100 * (partkey % 1000)) / 100.0
    price = np.round(qty * retail, 2)
    discount = rng.integers(0, 11, size=n) / 100.0
    tax = rng.integers(0, 9, size=n) / 100.0
    ar = rng.integers(0, 2, size=n, dtype=np.int64) * 2  # A=0 or R=2
    returnflag = np.where(receipt <= D_CURRENT, ar, 1).astype(np.int64)  # else N=1
    linestatus = (shipdate > D_CURRENT).astype(np.int64)  # O=1 else F=0
    return {"l_shipdate": shipdate, "l_returnflag": returnflag, "l_linestatus": linestatus,
            "l_quantity": qty, "l_extendedprice": price, "l_discount": discount, "l_tax": tax}


def lineitem_arrays(sf: float, seed: int = 42, rows: int | None = None, lo: int = 0,
                    hi: int | None = None) -> dict[str, np.ndarray]:
    """Appendix B lineitem generator (int64 dates/codes, float64 values).

    The table of ``rows`` rows (default 6e6 x SF) is generated in independently
    seeded chunks of LINEITEM_CHUNK rows, so any row range [lo, hi) -- one
    rank's shard -- is produced without generating the rest, and the shards of
    all ranks concatenate to the same table."""
    n = int(rows if rows is not None else round(6_000_000 * sf))
    hi = n if hi is None else min(int(hi), n)
    lo = max(0, int(lo))
    parts = []
    for c in range(lo // LINEITEM_CHUNK, (hi + LINEITEM_CHUNK - 1) // LINEITEM_CHUNK):
        c0 = c * LINEITEM_CHUNK
        full = _lineitem_chunk(sf, seed, c, min(LINEITEM_CHUNK, n - c0))
        a, b = max(lo, c0) - c0, min(hi, c0 + LINEITEM_CHUNK) - c0
        parts.append({k: v[a:b] for k, v in full.items()})
    if len(parts) == 1:
        return {k: np.ascontiguousarray(v) for k, v in parts[0].items()}
    if not parts:
        return {k: v[:0] for k, v in _lineitem_chunk(sf, seed, 0, 0).items()}
    return {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}


def lineitem_table(arrays: dict, columns=LINEITEM_COLUMNS):
    """Device table of the given lineitem arrays (numpy or torch)."""
    cols = []
    with trusted():
        for name in columns:
            v = Tensor(arrays[name])
            if name == "l_returnflag":
                cols.append(EncodedTensor(v, DictionaryEncoding(RETURNFLAG)))
            elif name == "l_linestatus":
                cols.append(EncodedTensor(v, DictionaryEncoding(LINESTATUS)))
            else:
                cols.append(plain(v))
    return table_from_columns(list(columns), cols)


# ---------------------------------------------------------------------------
# Q6: SUM(extendedprice * discount) over a 3-column range filter
# ---------------------------------------------------------------------------

Q6_SQL = ("SELECT SUM(rev) FROM (SELECT revenue(l_extendedprice, l_discount) FROM lineitem "
          "WHERE l_shipdate >= 8766 AND l_shipdate < 9131 AND l_discount >= 0.05 "
          "AND l_discount <= 0.07 AND l_quantity < 24)")


def q6_registry() -> UdfRegistry:
    reg = UdfRegistry()
    reg.register(UdfEntry("revenue", (("rev", FLOAT),), 2,
                          lambda p, d: (plain(mul(p.values, d.values)),), (), pe_outputs=False))
    return reg


# ---------------------------------------------------------------------------
# Q1: pricing summary, 4 groups x 8 aggregates
# ---------------------------------------------------------------------------

Q1_SQL = ("SELECT rf, ls, SUM(qty), SUM(price), SUM(disc_price), SUM(charge), AVG(qty), "
          "AVG(price), AVG(disc), COUNT(*) FROM (SELECT q1prep(l_returnflag, l_linestatus, "
          "l_quantity, l_extendedprice, l_discount, l_tax) FROM lineitem "
          "WHERE l_shipdate <= 10471) GROUP BY rf, ls")


def _q1prep(rf, ls, q, p, d, t):
    one = tensor(1.0)
    dp = mul(p.values, sub(one, d.values))
    ch = mul(dp, add(one, t.values))
    return (rf, ls, q, p, plain(dp), plain(ch), d)


def q1_registry() -> UdfRegistry:
    reg = UdfRegistry()
    reg.register(UdfEntry("q1prep", (("rf", STRING), ("ls", STRING), ("qty", FLOAT),
                                     ("price", FLOAT), ("disc_price", FLOAT), ("charge", FLOAT),
                                     ("disc", FLOAT)), 6, _q1prep, (), pe_outputs=False))
    return reg


def compile_sql(sql: str, catalog: Catalog, registry: UdfRegistry, trainable: bool = False):
    from .compiler import CompileConfig, compile_plan
    from .sql import bind, lower, parse

    return compile_plan(lower(bind(parse(sql), catalog, registry)),
                        CompileConfig(trainable=trainable), registry)


# ---------------------------------------------------------------------------
# Q3-style: customer |><| orders |><| lineitem, group by orderkey, top 10
# ---------------------------------------------------------------------------

MKTSEGMENT = StringDictionary(("AUTOMOBILE", "BUILDING", "FURNITURE", "HOUSEHOLD", "MACHINERY"))


def q3_arrays(sf: float, seed: int = 7) -> dict[str, dict[str, np.ndarray]]:
    """Appendix B Q3 tables: dbgen sparse order keys, customers without orders
    for custkey % 3 == 0, 1..7 lines per order."""
    rng = np.random.default_rng(seed)
    nc = max(3, int(round(150_000 * sf)))
    no = max(1, int(round(1_500_000 * sf)))
    cust = {"c_custkey": np.arange(1, nc + 1, dtype=np.int64),
            "c_mktsegment": rng.integers(0, 5, size=nc, dtype=np.int64)}
    i = np.arange(no, dtype=np.int64)
    okey = (i // 8) * 32 + i % 8 + 1
    ck = rng.integers(1, nc + 1, size=no, dtype=np.int64)
    ck = np.where(ck % 3 == 0, np.where(ck + 1 <= nc, ck + 1, ck - 1), ck)
    odate = rng.integers(D_1992_01_01, 10440 + 1, size=no, dtype=np.int64)
    orders = {"o_orderkey": okey, "o_custkey": ck, "o_orderdate": odate,
              "o_shippriority": np.zeros(no, dtype=np.int64)}
    lines = rng.integers(1, 8, size=no)
    lok = np.repeat(okey, lines)
    ldate = np.repeat(odate, lines) + rng.integers(1, 122, size=lok.size, dtype=np.int64)
    qty = rng.integers(1, 51, size=lok.size).astype(np.float64)
    pk = rng.integers(1, int(200_000 * max(sf, 1e-6)) + 1, size=lok.size, dtype=np.int64)
    retail = (90000 + (pk // 10) % 20001 + 100 * (pk % 1000)) / 100.0
    lineitem = {"l_orderkey": lok, "l_shipdate": ldate,
                "l_extendedprice": np.round(qty * retail, 2),
                "l_discount": rng.integers(0, 11, size=lok.size) / 100.0}
    return {"customer": cust, "orders": orders, "lineitem": lineitem}


def q3_catalog(tables: dict) -> Catalog:
    cat = Catalog()
    with trusted():
        c = tables["customer"]
        cat.register("customer", table_from_columns(
            ["c_custkey", "c_mktsegment"],
            [plain(Tensor(c["c_custkey"])),
             EncodedTensor(Tensor(c["c_mktsegment"]), DictionaryEncoding(MKTSEGMENT))]))
    for name in ("orders", "lineitem"):
        t = tables[name]
        cat.register(name, table_from_columns(list(t), [plain(Tensor(v)) for v in t.values()]))
    return cat


Q3_CUSTOMER = 'SELECT c_custkey FROM customer WHERE c_mktsegment = "BUILDING"'
Q3_ORDERS = ("SELECT o_orderkey, o_custkey, o_orderdate, o_shippriority FROM orders "
             "WHERE o_orderdate < 9204")
Q3_LINEITEM = ("SELECT l_orderkey, l_extendedprice, l_discount FROM lineitem "
               "WHERE l_shipdate > 9204")
Q3_TAIL = ("SELECT l_orderkey, SUM(rev), AVG(o_orderdate), AVG(o_shippriority) FROM "
           "(SELECT q3rev(l_orderkey, l_extendedprice, l_discount, o_orderdate, o_shippriority) "
           "FROM joined) GROUP BY l_orderkey ORDER BY sum_rev DESC LIMIT 10")


def q3_registry() -> UdfRegistry:
    from .storage import INT

    def q3rev(k, p, d, od, sp):
        return (k, plain(mul(p.values, sub(tensor(1.0), d.values))), od, sp)

    reg = UdfRegistry()
    reg.register(UdfEntry("q3rev", (("l_orderkey", INT), ("rev", FLOAT), ("o_orderdate", INT),
                                    ("o_shippriority", INT)), 5, q3rev, (), pe_outputs=False))
    return reg


class Q3Plan:
    """Compiled pieces of the Q3-style pipeline (the SQL subset has no JOIN:
    the three filters and the tail are SQL, the two equi-joins are
    kernels.equi_join)."""

    def __init__(self, catalog: Catalog):
        empty = UdfRegistry()
        self.cust = compile_sql(Q3_CUSTOMER, catalog, empty)
        self.orders = compile_sql(Q3_ORDERS, catalog, empty)
        self.lineitem = compile_sql(Q3_LINEITEM, catalog, empty)
        self.registry = q3_registry()
        self.tail = None
        from .replay import Pipeline

        # an unchanged catalog replays one CUDA graph of the whole plan
        self._pipeline = Pipeline(self.run_eager, ("customer", "orders", "lineitem"))

    def run(self, catalog: Catalog):
        return self._pipeline.run(catalog)

    def run_eager(self, catalog: Catalog):
        from .kernels import equi_join

        c = self.cust.run(catalog)
        o = self.orders.run(catalog)
        li = self.lineitem.run(catalog)
        # orders |><| BUILDING customers: keep o_orderkey, o_orderdate, o_shippriority
        oc = equi_join(list(o.columns), list(c.columns), 1, 0, left_out=[0, 2, 3], right_out=[])
        # lineitem |><| those orders: the tail reads these five columns only
        j = equi_join(list(li.columns), oc, 0, 0, right_out=[1, 2])
        names = ["l_orderkey", "l_extendedprice", "l_discount", "o_orderdate", "o_shippriority"]
        joined = table_from_columns(names, j)
        work = Catalog()
        work.register("joined", joined)
        if self.tail is None:
            self.tail = compile_sql(Q3_TAIL, work, self.registry)
        return self.tail.run(work)


# algorithmic bytes per row: each referenced base column once at 8 B
Q1_BYTES_PER_ROW = 56
Q6_BYTES_PER_ROW = 32

"""Golden results of random SQL queries, produced by running the REFERENCE.

Run in the build container (the reference is importable there, not on the
GPU host):

    python tests/golden/make_sql_golden.py

Two tables of one schema -- `t` (4 096 rows) and `u` (70 000 rows: the
hash / multi-CTA paths) -- with int64 keys of small, sparse and sorted-in-runs
ranges, a dictionary string column, float64 values that are multiples of 1/4
and float32 values i/100 (so every SUM / AVG is exact in any summation order
and results can be compared bit for bit), a wide int64 column, NaNs.  The
queries are drawn from the grammar the reference parses (tq/sql/parser.py):
filters (conjunctions of comparisons, NEP 50 literals, absent dictionary
strings), projections, GROUP BY one or two keys with COUNT / SUM / AVG,
global aggregates, ORDER BY [DESC] [LIMIT], subqueries, plus queries the
reference rejects (their exception class and message are recorded).
Writes tests/golden/sql_golden.npz and sql_golden.json; checked on the GPU by
tests/test_gpu_sql_golden.py.
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

import tensorquery as ref  # noqa: E402
from tensorquery.encodings import DictionaryEncoding, StringDictionary, plain  # noqa: E402
from tensorquery.tensor import Tensor  # noqa: E402

from sql_tables import FLOAT_COLS, INT_COLS, WORDS, mix_entry, tables as make_tables  # noqa: E402


def ref_table(cols: dict[str, np.ndarray]):
    enc = []
    for name, v in cols.items():
        if name == "s":
            enc.append(ref.EncodedTensor(Tensor(v), DictionaryEncoding(StringDictionary(WORDS))))
        else:
            enc.append(plain(Tensor(v)))
    return ref.table_from_columns(list(cols), enc)


def predicate(rg: random.Random) -> str:
    col = rg.choice(INT_COLS + FLOAT_COLS + ("s",))
    if col == "s":
        return f'{col} {rg.choice(["=", "<>"])} "{rg.choice(WORDS + ("plum",))}"'
    op = rg.choice(["=", "<>", "<", ">", "<=", ">="])
    # the lexer has no signed numbers: literals are >= 0
    lit = {"k1": lambda: rg.randint(0, 7), "k2": lambda: rg.choice([0, 1, 2, 2.5, 3.0]),
           "big": lambda: 5 + 1_000_000_007 * rg.randint(0, 300),
           "r": lambda: rg.randint(100, 7 * 3000), "v": lambda: rg.randint(0, 10**12),
           "f": lambda: rg.choice([0.0, 3.5, 10.25, 12, 49.75]),
           "g": lambda: rg.choice([0.05, 0.07, 0.0, 0.1, 1])}[col]()
    return f"{col} {op} {lit}"


def where(rg: random.Random) -> str:
    k = rg.choice([0, 0, 1, 1, 2, 3])
    return "" if k == 0 else " WHERE " + " AND ".join(predicate(rg) for _ in range(k))


def agg_items(rg: random.Random) -> list[tuple[str, str]]:
    """(SQL item, output name)"""
    out = [("COUNT(*)", "count")] if rg.random() < 0.7 else []
    for _ in range(rg.randint(1, 3)):
        func = rg.choice(["SUM", "AVG"])
        col = rg.choice(["k1", "k2", "v", "f", "g", "r"])
        item = (f"{func}({col})", f"{func.lower()}_{col}")
        if item not in out:
            out.append(item)
    return out


def order_limit(rg: random.Random, names: list[str]) -> str:
    names = [n for n in names if n != "count"]  # COUNT is a keyword, not an identifier
    s = ""
    if names and rg.random() < 0.5:
        s += f" ORDER BY {rg.choice(names)}" + (" DESC" if rg.random() < 0.5 else "")
    if rg.random() < 0.4:
        s += f" LIMIT {rg.choice([0, 1, 3, 10, 100000])}"
    return s


def gen_queries(rg: random.Random, count: int) -> list[str]:
    qs = []
    while len(qs) < count:
        tab = rg.choice(["t", "t", "u", "w"])
        kind = rg.choice(["proj", "group", "group", "group2", "global", "nested", "udf"])
        if kind == "proj":
            cols = rg.sample(list(INT_COLS + FLOAT_COLS + ("s",)), rg.randint(1, 3))
            tail = order_limit(rg, cols)
            if tab != "t" and "LIMIT" not in tail:  # keep the fixture small
                tail += " LIMIT 500"
            qs.append(f"SELECT {', '.join(cols)} FROM {tab}{where(rg)}{tail}")
        elif kind in ("group", "group2"):
            keys = rg.sample(["k1", "k2", "s", "big", "r"], 1 if kind == "group" else 2)
            aggs = agg_items(rg)
            items = keys + [a for a, _ in aggs]
            names = keys + [n for _, n in aggs]
            tail = order_limit(rg, names)
            if tab == "w" and "LIMIT" not in tail:  # keep the fixture small
                tail += " LIMIT 300"
            qs.append(f"SELECT {', '.join(items)} FROM {tab}{where(rg)} GROUP BY "
                      f"{', '.join(keys)}{tail}")
        elif kind == "udf":
            key = rg.choice(["k1", "s", "r", "big", "k2"])
            b = rg.choice(["k2", "f", "k1"])
            inner = f"SELECT mix({key}, f, {b}) FROM {tab}{where(rg)}"
            if rg.random() < 0.7:
                aggs = [a for a in ["COUNT(*)", "SUM(x)", "AVG(x)"] if rg.random() < 0.8] or ["SUM(x)"]
                names = ["k"] + [{"COUNT(*)": "count", "SUM(x)": "sum_x", "AVG(x)": "avg_x"}[a]
                                 for a in aggs]
                tail = order_limit(rg, names)
                if tab == "w" and "LIMIT" not in tail:
                    tail += " LIMIT 300"
                qs.append(f"SELECT k, {', '.join(aggs)} FROM ({inner}) GROUP BY k{tail}")
            else:
                qs.append(f"SELECT SUM(x), COUNT(*), AVG(x) FROM ({inner})")
        elif kind == "global":
            aggs = agg_items(rg)
            qs.append(f"SELECT {', '.join(a for a, _ in aggs)} FROM {tab}{where(rg)}")
        else:
            key = rg.choice(["k1", "s", "r", "big"])
            col = rg.choice(["v", "f", "k2"])
            inner = f"SELECT {key}, SUM({col}), COUNT(*) FROM {tab}{where(rg)} GROUP BY {key}"
            tail = order_limit(rg, [key, 'sum_' + col])
            if tab == "w" and "LIMIT" not in tail:
                tail += " LIMIT 300"
            outer = rg.choice([f"SELECT COUNT(*), SUM(sum_{col}), AVG(sum_{col}) FROM ({inner})",
                               f"SELECT {key}, sum_{col} FROM ({inner}) WHERE sum_{col} > 0{tail}"])
            qs.append(outer)
    return qs


REJECTED = [
    "SELECT k1 FROM t WHERE v > -5",                 # no signed literals in the lexer
    "SELECT k1, COUNT(*) FROM t GROUP BY k1 ORDER BY count",  # COUNT is a keyword
    "SELECT f, COUNT(*) FROM t GROUP BY f",          # float group key
    "SELECT SUM(s) FROM t",                          # SUM of a string column
    "SELECT nope FROM t",                            # unknown column
    "SELECT k1 FROM missing",                        # unknown table
    "SELECT k1 FROM t WHERE s < 3",                  # string vs number
    "SELECT k1, COUNT(*) FROM t GROUP BY k1 ORDER BY zz",
    "SELECT k1 FROM t LIMIT 2.5",
]


def main() -> None:
    rg = random.Random(20261017)
    tables = make_tables()
    cat = ref.Catalog()
    for name, cols in tables.items():
        cat.register(name, ref_table(cols))
    reg = ref.UdfRegistry()
    reg.register(mix_entry(ref))
    arrays: dict[str, np.ndarray] = {}
    # the tables are regenerated by the test (make_table, same seeds); their
    # checksums pin them
    sums = {f"{tn}/{cn}": hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()
            for tn, cols in tables.items() for cn, v in cols.items()}
    cases = []
    for qi, sql in enumerate(gen_queries(rg, 240) + REJECTED):
        case = {"sql": sql}
        try:
            plan = ref.lower(ref.bind(ref.parse(sql), cat, reg))
            out = ref.compile_plan(plan, ref.CompileConfig(), reg).run(cat)
            case["names"] = list(out.schema.names)
            case["rows"] = int(out.row_count)
            for ci, c in enumerate(out.columns):
                arrays[f"q{qi}/{ci}"] = np.asarray(c.values.data)
            case["dictionary"] = [c.is_dictionary() for c in out.columns]
        except Exception as e:  # the reference rejects it: record the error
            case["error"] = [type(e).__name__, str(e)]
        cases.append(case)
    np.savez_compressed(HERE / "sql_golden.npz", **arrays)
    (HERE / "sql_golden.json").write_text(json.dumps({"tables": sums, "cases": cases}, indent=1))
    ok = sum("error" not in c for c in cases)
    print(f"{len(cases)} queries: {ok} results, {len(cases) - ok} rejections")


if __name__ == "__main__":
    main()

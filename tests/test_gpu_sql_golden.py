"""Random SQL queries against the REFERENCE's own results
(tests/golden/make_sql_golden.py ran the reference on them): 160 queries --
filters, projections, one- and two-key GROUP BY with COUNT / SUM / AVG,
global aggregates, ORDER BY [DESC] [LIMIT], subqueries, an elementwise UDF
-- over 4 096-, 70 000- and 400 000-row tables, each in the reference's
storage widths and in compact storage (dense, sparse, sorted-in-runs and dictionary keys; the
fused scan, hash / bitmap / runs group-by, top-k and sort paths), compared
bit for bit (every float64 sum in the fixture is exact in any order; float32
global aggregates, summed in float32 like the reference, within a few ulps),
and 9 queries the reference rejects, compared by exception class and
message."""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200.encodings import DictionaryEncoding, StringDictionary

G = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(G))
from sql_tables import WORDS, mix_entry, tables  # noqa: E402

META = json.loads((G / "sql_golden.json").read_text())
CASES = META["cases"]


def test_sql_golden_tables_reproduce():
    """The tables the fixture was made from are rebuilt bit for bit (CPU)."""
    for tn, cols in tables().items():
        for cn, v in cols.items():
            h = hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()
            assert h == META["tables"][f"{tn}/{cn}"], (tn, cn)


def _catalog(compact: bool = False):
    from paper_2211_02753_b200 import compact as cp

    cat = tq.Catalog()
    for name, cols in tables().items():
        enc = []
        with tq.encodings.trusted():
            for cn, v in cols.items():
                if cn == "s":
                    enc.append(tq.EncodedTensor(tq.Tensor(v),
                                                DictionaryEncoding(StringDictionary(WORDS))))
                else:
                    enc.append(tq.plain(tq.Tensor(v)))
        table = tq.table_from_columns(list(cols), enc)
        cat.register(name, cp.compact_table(table) if compact else table)
    return cat


@pytest.fixture(scope="module", params=["wide", "compact"])
def catalog(request):
    """The reference's storage widths, and the same tables in compact
    storage (narrow integers, scaled decimals, uint8 codes):
    every query must give the reference's result on both."""
    return _catalog(request.param == "compact")


@pytest.fixture(scope="module")
def arrays():
    return np.load(G / "sql_golden.npz")


@pytest.mark.gpu
@pytest.mark.parametrize("qi", range(len(CASES)))
def test_sql_query_matches_reference(qi, catalog, arrays):
    case = CASES[qi]
    reg = tq.UdfRegistry()
    reg.register(mix_entry(tq))
    if "error" in case:
        with pytest.raises(Exception) as ei:
            tq.compile_plan(tq.lower(tq.bind(tq.parse(case["sql"]), catalog, reg)),
                            tq.CompileConfig(), reg).run(catalog)
        assert [type(ei.value).__name__, str(ei.value)] == case["error"], case["sql"]
        return
    q = tq.compile_plan(tq.lower(tq.bind(tq.parse(case["sql"]), catalog, reg)),
                        tq.CompileConfig(), reg)
    # eager (recording) run, capturing run, CUDA-graph replay: all three
    # results must be the reference's
    for _ in range(3):
        _check(case, q.run(catalog), arrays, qi)


def _check(case, out, arrays, qi):
    assert list(out.schema.names) == case["names"], case["sql"]
    assert out.row_count == case["rows"], case["sql"]
    for ci, col in enumerate(out.columns):
        exp = arrays[f"q{qi}/{ci}"]
        got = col.values.numpy()
        assert col.is_dictionary() == case["dictionary"][ci], case["sql"]
        assert got.dtype == exp.dtype, (case["sql"], ci, got.dtype, exp.dtype)
        assert got.shape == exp.shape, (case["sql"], ci)
        if exp.dtype.kind == "f":  # NaNs by position (payloads may differ)
            nan = np.isnan(exp)
            assert np.array_equal(np.isnan(got), nan), (case["sql"], ci)
            got, exp = got[~nan], exp[~nan]
        if exp.dtype == np.float32:
            # a float32 global SUM / AVG accumulates in float32 like the
            # reference (input-dtype sum), whose numpy reduction adds
            # pairwise: the last bit depends on the order (a few ulps)
            np.testing.assert_allclose(got, exp, rtol=4e-7, atol=0, err_msg=case["sql"])
            continue
        assert got.tobytes() == exp.tobytes(), (case["sql"], ci, got[:8], exp[:8])

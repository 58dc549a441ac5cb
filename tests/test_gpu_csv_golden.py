"""read_csv on 120 generated >= 64 KB files against the REFERENCE's own
results (tests/golden/make_csv_golden.py ran tensorquery.storage.read_csv):
quoting, escaped quotes, embedded separators and newlines, CRLF, whitespace,
signs, exponents, inf / nan, underscores and Unicode digits (Python's int()
/ float() accept them), subnormals, overflow, empty cells, short rows.  A
table must equal the reference's column for column (values by checksum,
dictionaries entry for entry); an error must carry the reference's class and
message (line numbers included)."""

from __future__ import annotations

import io
import json
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2211_02753_b200 import csvdev
from paper_2211_02753_b200.storage import ColumnType, Schema, read_csv

G = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(G))
from csv_cases import case_text, column_digest  # noqa: E402

CASES = json.loads((G / "csv_golden.json").read_text(encoding="utf-8"))["cases"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[f"seed{c['seed']}" for c in CASES])
def test_read_csv_matches_reference(case):
    text, schema = case_text(case["seed"])
    sch = Schema(tuple((n, ColumnType(k)) for n, k in schema))
    assert len(text.encode("utf-8")) >= csvdev.DEVICE_CSV_MIN_BYTES
    if "error" in case:
        with pytest.raises(Exception) as ei:
            read_csv(io.StringIO(text, newline=""), sch)
        assert [type(ei.value).__name__, str(ei.value)] == case["error"]
        return
    t = read_csv(io.StringIO(text, newline=""), sch)
    assert len(t.columns) == len(case["columns"])
    for c, exp in zip(t.columns, case["columns"]):
        v = c.values.numpy()
        assert str(v.dtype) == exp["dtype"] and v.shape[0] == exp["rows"]
        assert column_digest(v) == exp["digest"]
        if "dictionary" in exp:
            assert c.is_dictionary()
            assert list(c.encoding.dictionary.entries) == exp["dictionary"]

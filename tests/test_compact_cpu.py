"""CPU: host logic of compact storage -- the rewrite of float64 predicates on a
scaled-decimal column into exact int64 comparisons on the stored integers
(lazy.decimal_predicates), checked against numpy's float64 comparison of the
decoded values for every stored integer in a range, and the decode-expression
shape the scan kernel and the filter rewrite recognise."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2211_02753_b200 import _native as nat
from paper_2211_02753_b200.compact import decode_expr
from paper_2211_02753_b200.lazy import compact_source, decimal_predicates

OPS = {"=": np.equal, "<>": np.not_equal, "<": np.less, ">": np.greater, "<=": np.less_equal,
       ">=": np.greater_equal}
CMP = {"=": np.equal, "<>": np.not_equal, "<": np.less, ">": np.greater, "<=": np.less_equal,
       ">=": np.greater_equal}


def _apply(preds, c: np.ndarray) -> np.ndarray:
    keep = np.ones(c.shape, dtype=bool)
    for op, cmp, li in preds:
        if cmp == nat.CMP_NONE:
            keep &= False
        elif cmp == nat.CMP_ALL:
            pass
        else:
            assert cmp == nat.CMP_I64
            keep &= CMP[op](c, np.int64(li))
    return keep


@pytest.mark.parametrize("divisor", [1, 10, 100, 10000])
def test_decimal_predicates_match_float_compare(divisor):
    c = np.arange(-3000, 3001, dtype=np.int64)
    values = c / divisor  # numpy true division: correctly rounded, what is stored
    lits = [0.0, 0.05, 0.07, -0.005, 0.1, 1.0, 3, -2, 0.3, 29.99, -29.995, 1e300, -1e300,
            float("inf"), float("-inf"), float("nan"), 5e-324, 0.015, 12.345]
    for lit in lits:
        for op, f in OPS.items():
            preds = decimal_predicates(op, float(lit), divisor)
            exp = f(values, np.float64(lit))
            got = _apply(preds, c)
            np.testing.assert_array_equal(got, exp, err_msg=f"{op} {lit} /{divisor}")


def test_decode_expression_shapes():
    stored = torch.zeros(4, dtype=torch.int16)
    e = decode_expr(stored, 100)
    assert e.op == "decimal" and e.dtype == "float64"
    assert compact_source(e) == (stored, 100)
    i = decode_expr(torch.zeros(3, dtype=torch.uint8), 0)
    assert i.op == "cast" and i.dtype == "int64"
    src = compact_source(i)
    assert src is not None and src[1] == 0 and src[0].dtype == torch.uint8

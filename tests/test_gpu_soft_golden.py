"""Trainable (soft) queries against the REFERENCE's own results
(tests/golden/make_soft_golden.py ran the reference): soft COUNT / SUM / AVG
grouped by one or two probability-encoded keys (softmax heads and one-hot
bags, both key orders), soft global aggregates over a score UDF with and
without a filter -- on four shapes; the outputs and the tape gradients of
every model parameter for a seeded random loss over the outputs (float64
models: outputs rtol 1e-9 + the fixed-point count grid's n 2^-31, gradients
rtol 1e-7)."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2211_02753_b200 as tq

G = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(G))
from soft_cases import run_case  # noqa: E402

CASES = json.loads((G / "soft_golden.json").read_text())["cases"]


@pytest.fixture(scope="module")
def arrays():
    return np.load(G / "soft_golden.npz")


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c["tag"] for c in CASES])
def test_soft_query_matches_reference(case, arrays):
    names, outs, grads = run_case(tq, case["sql"], tuple(case["shape"]),
                                  lambda g: g.data.detach().cpu().numpy())
    assert names == case["names"], case["sql"]
    # soft counts over one-hot x dense keys accumulate probabilities in a
    # 2^-30 fixed-point shared-memory grid (error <= n 2^-31 per
    # cell); everything else is float64 arithmetic
    n = case["shape"][0]
    for j, got in enumerate(outs):
        exp = arrays[f"{case['tag']}/out{j}"]
        assert got.shape == exp.shape, (case["sql"], j)
        if exp.dtype.kind == "f":
            np.testing.assert_allclose(got, exp, rtol=1e-9, atol=n * 2.0**-31,
                                       err_msg=case["sql"])
        else:
            np.testing.assert_array_equal(got, exp, err_msg=case["sql"])
    assert sorted(grads) == case["grads"], case["sql"]
    for pn, g in grads.items():
        np.testing.assert_allclose(g, arrays[f"{case['tag']}/grad/{pn}"], rtol=1e-7, atol=1e-9,
                                   err_msg=f"{case['sql']} d{pn}")

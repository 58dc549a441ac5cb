"""GPU parity of the differentiable path (soft group-by, softmax, LLP step).

Gradients and soft grids: rtol 1e-5 against the float64 oracle (north-star
tolerance for LLP gradients); float64 inputs are compared at 1e-10.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import relational as orc
import paper_2211_02753_b200 as tq
from paper_2211_02753_b200 import kernels as K
from paper_2211_02753_b200.tensor import Tape, backward, reduce_sum, mul

pytestmark = pytest.mark.gpu


def _pe(rng, n, k, dtype="float64"):
    logits = rng.normal(size=(n, k))
    return orc.softmax(logits).astype(dtype), logits


def test_spec_soft_count_examples():
    p = tq.EncodedTensor(tq.tensor([[0.9, 0.1], [0.2, 0.8], [0.7, 0.3]]),
                         tq.ProbabilityEncoding(2))
    # count grids accumulate in 2^-30 fixed point per CTA: |error| <= 2^-31 per row
    np.testing.assert_allclose(tq.soft_count(p).numpy(), [1.8, 1.2], rtol=0, atol=3 * 2.0**-31)
    oh = tq.one_hot_pe([0, 1, 0], 2)
    np.testing.assert_array_equal(tq.soft_count(oh).numpy(), [2, 1])
    half = tq.EncodedTensor(tq.tensor([[0.5, 0.5]]), tq.ProbabilityEncoding(2))
    g = tq.soft_groupby([half, half]).counts.numpy()
    np.testing.assert_allclose(g, [[0.25, 0.25], [0.25, 0.25]])


@pytest.mark.parametrize("agg", ["count", "sum", "avg"])
def test_soft_groupby_forward_backward(agg):
    rng = np.random.default_rng(21)
    n = 5000
    p1, _ = _pe(rng, n, 3)
    p2, _ = _pe(rng, n, 4)
    vals = rng.normal(size=n)
    G = rng.normal(size=(3, 4))
    exp = orc.soft_groupby([p1, p2], agg, vals if agg != "count" else None)
    with Tape() as tape:
        a = tq.Tensor(p1)
        b = tq.Tensor(p2)
        v = tq.Tensor(vals)
        pa = tq.EncodedTensor(a, tq.ProbabilityEncoding(3))
        pb = tq.EncodedTensor(b, tq.ProbabilityEncoding(4))
        res = tq.soft_groupby([pa, pb], agg, v if agg != "count" else None)
        # counts: fixed-point accumulation, |error| <= n * 2^-31; sum/avg: float64
        np.testing.assert_allclose(res.counts.numpy(), exp, rtol=1e-10, atol=n * 2.0**-31)
        loss = reduce_sum(mul(res.counts, tq.tensor(G)))
        backward(loss)
        ga, gb, gv = tape.gradient(a), tape.gradient(b), tape.gradient(v)
    if agg == "count":
        (ea, eb), _ = orc.soft_groupby_vjp([p1, p2], G)
        np.testing.assert_allclose(ga.numpy(), ea, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(gb.numpy(), eb, rtol=1e-10, atol=1e-12)
    elif agg == "sum":
        (ea, eb), ev = orc.soft_groupby_vjp([p1, p2], G, vals)
        np.testing.assert_allclose(ga.numpy(), ea, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(gv.numpy(), ev, rtol=1e-10, atol=1e-12)
    else:
        assert ga is not None and gb is not None and gv is not None


def test_onehot_times_dense_llp_shape():
    rng = np.random.default_rng(22)
    n, bags = 20_000, 1000
    p, logits = _pe(rng, n, 2, "float32")
    codes = rng.integers(0, bags, size=n)
    exp = orc.soft_groupby([orc.one_hot(codes, bags), p.astype(np.float64)])
    pe = tq.EncodedTensor(tq.Tensor(p), tq.ProbabilityEncoding(2))
    bag = tq.one_hot_pe(codes, bags)
    got = tq.soft_groupby([bag, pe]).counts
    assert got.dtype == "float64"  # one_hot_pe default float64 promotes the grid
    np.testing.assert_allclose(got.numpy(), exp, rtol=1e-5, atol=1e-6)


def test_softmax_and_pe_decode():
    rng = np.random.default_rng(23)
    for k in (2, 7, 1000):
        logits = rng.normal(size=(777, k))
        logits[0, :] = 0.0  # ties -> lowest class
        pe = tq.pe_encode(tq.Tensor(logits))
        np.testing.assert_allclose(pe.values.numpy(), orc.softmax(logits), rtol=1e-12, atol=1e-15)
        codes = tq.pe_decode(pe).values.numpy()
        np.testing.assert_array_equal(codes, orc.pe_decode(orc.softmax(logits)))
        g = rng.normal(size=(777, k))
        with Tape() as tape:
            x = tq.Tensor(logits)
            y = tq.pe_encode(x).values
            backward(reduce_sum(mul(y, tq.tensor(g))))
            dx = tape.gradient(x).numpy()
        np.testing.assert_allclose(dx, orc.softmax_vjp(orc.softmax(logits), g), rtol=1e-9, atol=1e-12)


def test_pe_validation_errors():
    with pytest.raises(tq.EncodingError, match="lie in"):
        tq.EncodedTensor(tq.tensor([[1.5, -0.5]]), tq.ProbabilityEncoding(2))
    with pytest.raises(tq.EncodingError, match="sum to 1"):
        tq.EncodedTensor(tq.tensor([[0.5, 0.4]]), tq.ProbabilityEncoding(2))
    # NaN rows pass the reference's max-based checks
    tq.EncodedTensor(tq.tensor([[np.nan, 0.5]]), tq.ProbabilityEncoding(2))
    with pytest.raises(tq.EncodingError):
        tq.one_hot_pe([0, 3], 3)

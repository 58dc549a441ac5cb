"""GPU: the streaming skinny-linear kernels (tdp_linear_fwd / tdp_linear_wgrad)
behind Linear layers of trainable-query models, against float64 torch.

float64 inputs: rtol 1e-12; float32 inputs: rtol 1e-5 on the forward (float32
accumulation over d terms, like BLAS) and 1e-5 on gradients (float64
accumulation over rows).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200.autograd import LINEAR_MIN_ROWS, linear_eligible
from paper_2211_02753_b200.tensor import Tape, backward, linear, mul, reduce_sum

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("d,k", [(64, 2), (7, 1), (33, 3), (256, 8), (100, 5)])
def test_linear_forward_and_gradients(dtype, d, k):
    rng = np.random.default_rng(d * 10 + k)
    n = LINEAR_MIN_ROWS + 12345
    X = rng.normal(size=(n, d)).astype(dtype)
    W = rng.normal(size=(d, k)).astype(dtype)
    b = rng.normal(size=k).astype(dtype)
    G = rng.normal(size=(n, k))
    x = tq.Tensor(X)
    assert linear_eligible(x.data, tq.Tensor(W).data)
    with Tape() as tape:
        w, bb = tq.Tensor(W), tq.Tensor(b)
        y = linear(x, w, bb)
        backward(reduce_sum(mul(y, tq.tensor(G, dtype=dtype))))
        dw, db = tape.gradient(w).numpy(), tape.gradient(bb).numpy()
    X64, W64 = X.astype(np.float64), W.astype(np.float64)
    exp = X64 @ W64 + b.astype(np.float64)
    rtol = 1e-12 if dtype == "float64" else 1e-5
    atol = 1e-12 if dtype == "float64" else 1e-4
    np.testing.assert_allclose(y.numpy(), exp, rtol=rtol, atol=atol)
    g = G.astype(dtype).astype(np.float64)
    # float32 inputs: per-stage float32 partial sums (<= 32 rows) folded into
    # float64; bound relative to sum |x||g| (cancellation-safe)
    eps = 2e-6 if dtype == "float32" else 1e-13
    scale = np.abs(X64).T @ np.abs(g)
    assert np.all(np.abs(dw - X64.T @ g) <= eps * scale + 1e-12)
    assert np.all(np.abs(db - g.sum(axis=0)) <= eps * np.abs(g).sum(axis=0) + 1e-12)

"""GPU: the fused soft count over a linear head (tdp_soft_linear_count_fwd/bwd)
-- soft_groupby(one_hot keys x pe_encode(linear(X))) in one pass over X --
against float64 torch and against the composed kernels.

Tolerances: the count grid is the fixed-point sum of float32 (or float64)
probabilities: rtol 1e-5 + atol n * 2^-31 against float64; bit-identical to
the composed path (same per-row arithmetic).  dW / db: float32 row partials
folded into float64, bound eps * sum |x| |dz| with eps 1e-5 (float32) /
1e-12 (float64).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200.autograd import LINEAR_MIN_ROWS
from paper_2211_02753_b200.tensor import (Tape, backward, linear, mark_constant, mul, pending_softmax,
                                          reduce_sum, reshape)

pytestmark = pytest.mark.gpu


def _reference(X, W, b, codes_list, ks, dense_pos, G):
    """float64 torch: grid and (dW, db) of sum(grid * G)."""
    X, W, b = (torch.as_tensor(a, dtype=torch.float64, device="cuda") for a in (X, W, b))
    W.requires_grad_(True)
    b.requires_grad_(True)
    P = torch.softmax(X @ W + b, dim=1)
    n, k = P.shape
    cells = int(np.prod(ks))
    strides = [int(np.prod(ks[j + 1:])) for j in range(len(ks))]
    base = torch.zeros(n, dtype=torch.int64, device="cuda")
    it = iter(codes_list)
    for j, kj in enumerate(ks):
        if j != dense_pos:
            base += torch.as_tensor(next(it), device="cuda") * strides[j]
    idx = base[:, None] + torch.arange(k, device="cuda")[None, :] * strides[dense_pos]
    grid = torch.zeros(cells, dtype=torch.float64, device="cuda").index_add(0, idx.reshape(-1),
                                                                           P.reshape(-1))
    (grid * torch.as_tensor(G, device="cuda")).sum().backward()
    return grid.detach().cpu().numpy(), W.grad.cpu().numpy(), b.grad.cpu().numpy(), P.detach()


def _run(X, W, b, codes_list, ks, dense_pos, G, dtype, fuse=True):
    k = W.shape[1]
    with Tape() as tape:
        x = mark_constant(tq.Tensor(X))
        w, bb = tq.Tensor(W), tq.Tensor(b)
        pe = tq.pe_encode(linear(x, w, bb))
        if fuse:
            assert pending_softmax(pe.values) is not None
        else:
            pe.values.data  # materialise: composed kernels
        keys, it = [], iter(codes_list)
        for j, kj in enumerate(ks):
            keys.append(pe if j == dense_pos else tq.one_hot_pe(torch.as_tensor(next(it)), kj))
        res = tq.soft_groupby(keys)
        if fuse:
            assert pending_softmax(pe.values) is not None, "fused path not taken"
        grid = res.counts
        backward(reduce_sum(mul(reshape_flat(grid), tq.tensor(G, dtype=grid.dtype))))
        return grid.numpy().reshape(-1), tape.gradient(w).numpy(), tape.gradient(bb).numpy()


def reshape_flat(t):
    return reshape(t, (t.size,))


CASES = [
    # dtype, d, k, one-hot key sizes (dense inserted at dense_pos), dense_pos
    ("float32", 64, 2, (1000,), 1),
    ("float32", 32, 3, (37, 5), 0),
    ("float32", 64, 5, (11,), 1),
    ("float32", 32, 8, (100,), 0),
    ("float64", 32, 2, (250,), 1),
    ("float64", 32, 4, (7, 3), 2),
    # strided feature layout (d not 32 / 64, a multiple of 4)
    ("float32", 100, 2, (1000,), 1),
    ("float32", 36, 3, (37, 5), 0),
    ("float32", 92, 4, (9,), 0),
    ("float64", 20, 1, (30,), 1),
    ("float64", 44, 1, (30,), 0),
]


def _contiguous(dtype, d):
    return d in ((32, 64) if dtype == "float32" else (32,))


@pytest.mark.parametrize("dtype,d,k,oh,dense_pos", CASES)
def test_fused_soft_linear_count(dtype, d, k, oh, dense_pos):
    rng = np.random.default_rng(d * 100 + k)
    n = LINEAR_MIN_ROWS + 4321  # ragged tail stage
    X = rng.normal(size=(n, d)).astype(dtype)
    W = (rng.normal(size=(d, k)) * 0.3).astype(dtype)
    b = rng.normal(size=k).astype(dtype)
    codes = [rng.integers(0, kj, size=n) for kj in oh]
    ks = list(oh)
    ks.insert(dense_pos, k)
    G = rng.normal(size=int(np.prod(ks)))
    grid, dw, db = _run(X, W, b, codes, ks, dense_pos, G, dtype)
    rgrid, rdw, rdb, P = _reference(X, W, b, codes, ks, dense_pos, G)
    np.testing.assert_allclose(grid, rgrid, rtol=1e-5, atol=n * 2.0**-31)
    # gradient bound: eps * sum_i |x_i| |dz_i|
    Pn = P.cpu().numpy()
    eps = 1e-5 if dtype == "float32" else 1e-12
    strides = [int(np.prod(ks[j + 1:])) for j in range(len(ks))]
    base = np.zeros(n, dtype=np.int64)
    it = iter(codes)
    for j in range(len(ks)):
        if j != dense_pos:
            base += next(it) * strides[j]
    g = G[base[:, None] + np.arange(k)[None, :] * strides[dense_pos]]
    dz = Pn * (g - (Pn * g).sum(axis=1, keepdims=True))
    scale = np.abs(X.astype(np.float64)).T @ np.abs(dz)
    assert np.all(np.abs(dw - rdw) <= eps * scale + 1e-9), np.max(np.abs(dw - rdw) / (scale + 1e-30))
    assert np.all(np.abs(db - rdb) <= eps * np.abs(dz).sum(axis=0) + 1e-9)
    # the composed kernels give the identical grid (same row arithmetic in the
    # contiguous layout; the strided layout sums the row dots in another
    # order) and matching gradients
    cgrid, cdw, cdb = _run(X, W, b, codes, ks, dense_pos, G, dtype, fuse=False)
    onepass = dtype == "float32" and k == 2 and len(oh) == 1 and d in (32, 64)
    if onepass:  # llp_onepass.cu: float64 sums of the probabilities, not 2^-30 fixed point
        np.testing.assert_allclose(grid, cgrid, rtol=1e-8, atol=n * 2.0**-31)
    elif _contiguous(dtype, d):
        np.testing.assert_array_equal(grid, cgrid)
    else:
        np.testing.assert_allclose(grid, cgrid, rtol=1e-6 if dtype == "float32" else 1e-13,
                                   atol=n * 2.0**-31)
    assert np.all(np.abs(dw - cdw) <= 2 * eps * scale + 1e-9)


def test_pending_linear_materialises_like_eager():
    rng = np.random.default_rng(5)
    n, d, k = LINEAR_MIN_ROWS + 77, 64, 2
    X = rng.normal(size=(n, d)).astype("float32")
    W = rng.normal(size=(d, k)).astype("float32")
    b = rng.normal(size=k).astype("float32")
    x = mark_constant(tq.Tensor(X))
    y = linear(x, tq.Tensor(W), tq.Tensor(b))
    assert y.is_lazy and y.shape == (n, k) and y.dtype == "float32"
    np.testing.assert_allclose(y.numpy(), X.astype(np.float64) @ W + b, rtol=1e-5, atol=1e-4)
    p = tq.pe_encode(linear(x, tq.Tensor(W), tq.Tensor(b)))
    ref = torch.softmax(torch.as_tensor(X @ W + b, device="cuda"), 1).cpu().numpy()
    np.testing.assert_allclose(p.values.numpy(), ref, rtol=1e-5, atol=1e-6)
    # non-count soft aggregates use the composed path
    w8 = tq.Tensor(rng.normal(size=n))
    with Tape():
        pe = tq.pe_encode(linear(x, tq.Tensor(W), tq.Tensor(b)))
        s = tq.soft_groupby([pe], "sum", w8)
        exp = (ref * w8.numpy()[:, None]).sum(axis=0)
        np.testing.assert_allclose(s.counts.numpy(), exp, rtol=1e-5)


def test_unsupported_shapes_fall_back():
    rng = np.random.default_rng(9)
    n, d, k = LINEAR_MIN_ROWS + 5, 50, 2  # d not a multiple of 4
    X = rng.normal(size=(n, d)).astype("float32")
    W = rng.normal(size=(d, k)).astype("float32")
    b = np.zeros(k, dtype="float32")
    codes = rng.integers(0, 9, size=n)
    with Tape() as tape:
        x = mark_constant(tq.Tensor(X))
        w = tq.Tensor(W)
        pe = tq.pe_encode(linear(x, w, tq.Tensor(b)))
        assert pending_softmax(pe.values) is None
        res = tq.soft_groupby([tq.one_hot_pe(torch.as_tensor(codes), 9), pe])
        backward(reduce_sum(res.counts))
        assert tape.gradient(w) is not None
    P = torch.softmax(torch.as_tensor(X.astype(np.float64) @ W), 1).numpy()
    exp = np.zeros((9, k))
    np.add.at(exp, codes, P)
    np.testing.assert_allclose(res.counts.numpy(), exp, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("with_bag", [False, True])
def test_wide_head_chunked_soft_count_equals_unfused(dtype, with_bag, monkeypatch):
    """A wide head (SURVEY 4': Linear(d, K) with K large) whose logits would not
    fit is counted in row chunks (autograd._ChunkedSoftLinearCount): the grid
    and the tape gradients equal the materialised (unfused) path's."""
    from paper_2211_02753_b200 import autograd as AG
    from paper_2211_02753_b200.tensor import Tape, backward, mul, reduce_sum

    rng = np.random.default_rng(5)
    n, d, k, bags = 5000, 16, 300, 6
    X = rng.normal(size=(n, d)).astype(dtype)
    codes = rng.integers(0, bags, size=n)
    G = rng.normal(size=(bags, k) if with_bag else (k,))

    def run(wide: bool):
        monkeypatch.setattr(AG, "WIDE_HEAD_BYTES", 0 if wide else 1 << 62)
        monkeypatch.setattr(AG, "CHUNK_BYTES", 64 << 10)  # ~13-27 rows x 300 per chunk
        lin = tq.Linear(d, k, np.random.default_rng(9), name="w", dtype=dtype)
        with Tape() as tape:
            pe = tq.pe_encode(lin(mark_constant(tq.Tensor(X))))  # a catalog column
            keys = [tq.one_hot_pe(codes, bags), pe] if with_bag else [pe]
            grid = tq.soft_groupby(keys).counts
            backward(reduce_sum(mul(grid, tq.tensor(G.astype(dtype)))))
            return (grid.numpy(), tape.gradient(lin.weight.value).numpy(),
                    tape.gradient(lin.bias.value).numpy())

    from paper_2211_02753_b200 import kernels as K

    calls = [0]
    real = K.chunked_soft_linear_count

    def counted(*a, **kw):
        calls[0] += 1
        return real(*a, **kw)

    monkeypatch.setattr(K, "chunked_soft_linear_count", counted)
    gw, dww, dbw = run(True)
    assert calls[0] == 1  # the chunked path ran
    gu, dwu, dbu = run(False)
    assert calls[0] == 1
    tol = 1e-9 if dtype == "float64" else 2e-5
    np.testing.assert_allclose(gw, gu, rtol=tol, atol=n * 2.0**-31)
    np.testing.assert_allclose(dww, dwu, rtol=tol, atol=tol * np.abs(dwu).max())
    np.testing.assert_allclose(dbw, dbu, rtol=tol, atol=tol * np.abs(dbu).max())

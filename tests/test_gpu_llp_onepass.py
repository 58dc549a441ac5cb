"""GPU: the one-pass LLP step (csrc/llp_onepass.cu) against a
float64 recompute of the reference tape's closed forms and against the
two-pass kernels (TDP_LLP_ONEPASS=0): count grid, dW, db at rtol 1e-5 of the
float64 values (north_star's LLP-gradient tolerance)."""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200.storage import tensor_type
from paper_2211_02753_b200.tensor import backward
from paper_2211_02753_b200.training import mse_loss, prediction_vector

pytestmark = pytest.mark.gpu


def _f64_reference(X, bag, W, b, target, bags, bag_first):
    Xd = X.double()
    P = torch.softmax(Xd @ W.double() + b.double(), dim=1)
    grid = torch.zeros((bags, 2), dtype=torch.float64, device=X.device)
    grid.index_add_(0, bag, P)
    flat = grid.reshape(-1) if bag_first else grid.t().reshape(-1)
    G = 2.0 * (flat - target) / flat.numel()
    G2 = G.view(bags, 2) if bag_first else G.view(2, bags).t()
    g = G2[bag]
    dZ = P * (g - (P * g).sum(dim=1, keepdim=True))
    return flat, Xd.t() @ dZ, dZ.sum(dim=0)


def _engine_step(X, bag, bags, target, bag_first, seed=0):
    d = X.shape[1]
    model = tq.Linear(d, 2, np.random.default_rng(seed), name="lin")
    bag_pe = tq.one_hot_pe(bag, bags)
    reg = tq.UdfRegistry()
    if bag_first:
        schema = (("Bag", tensor_type(bags)), ("Pred", tensor_type(2)))
        body = lambda c: (bag_pe, tq.pe_encode(model(c.values)))  # noqa: E731
        sql = "SELECT Bag, Pred, COUNT(*) FROM llp(T) GROUP BY Bag, Pred"
    else:
        schema = (("Pred", tensor_type(2)), ("Bag", tensor_type(bags)))
        body = lambda c: (tq.pe_encode(model(c.values)), bag_pe)  # noqa: E731
        sql = "SELECT Pred, Bag, COUNT(*) FROM llp(T) GROUP BY Pred, Bag"
    reg.register(tq.UdfEntry("llp", schema, 1, body, model.parameters))
    cat = tq.Catalog()
    cat.register_tensor(tq.Tensor(X), "T")
    q = tq.compile_plan(tq.lower(tq.bind(tq.parse(sql), cat, reg)),
                        tq.CompileConfig(trainable=True), reg)
    res = q.run(cat)
    pred = prediction_vector(res, q)
    loss = mse_loss(pred, tq.Tensor(target))
    backward(loss)
    grads = {p.name: q.tape.gradient(p.value).data.clone() for p in q.parameters()}
    grid = pred.data.detach().clone()
    q.end_session()
    return grid, grads["lin.weight"], grads["lin.bias"], model


def _rel(a, b):
    return float((a.double() - b).abs().max() / b.abs().max().clamp_min(1e-300))


@pytest.mark.parametrize("n,d,bags,bag_first", [(300_001, 64, 1000, True), (200_000, 32, 37, False),
                                                (150_000, 64, 5000, True)])
def test_onepass_llp_step_matches_float64_and_two_pass(n, d, bags, bag_first, monkeypatch):
    g = torch.Generator(device="cuda").manual_seed(n)
    X = torch.randn(n, d, generator=g, device="cuda")
    bag = torch.randint(0, bags, (n,), generator=g, device="cuda")
    bag[bag == 3] = 4  # an empty bag
    target = torch.rand(bags * 2, generator=g, device="cuda", dtype=torch.float64) * (n / bags)
    monkeypatch.setenv("TDP_LLP_ONEPASS", "1")
    grid1, dW1, db1, model = _engine_step(X, bag, bags, target, bag_first)
    grid1b, dW1b, db1b, _ = _engine_step(X, bag, bags, target, bag_first)
    assert torch.equal(grid1, grid1b) and torch.equal(dW1, dW1b)  # bitwise repeatable
    monkeypatch.setenv("TDP_LLP_ONEPASS", "0")
    grid2, dW2, db2, _ = _engine_step(X, bag, bags, target, bag_first)
    W, b = model.weight.value.data, model.bias.value.data
    rgrid, rdW, rdb = _f64_reference(X, bag, W, b, target, bags, bag_first)
    for got in (grid1, grid2):
        assert _rel(got, rgrid) < 1e-6  # float32 logits: ~1e-8
    for got, ref in ((dW1, rdW), (db1, rdb), (dW2, rdW), (db2, rdb)):
        assert _rel(got, ref) < 1e-5, (_rel(got, ref))


def test_onepass_bag_index_is_cached_and_invalidated():
    from paper_2211_02753_b200.autograd import bag_index

    codes = torch.randint(0, 50, (100_000,), device="cuda")
    p1, o1 = bag_index(codes, 50)
    p2, o2 = bag_index(codes, 50)
    assert p1 is p2 and o1 is o2
    assert torch.equal(codes[p1.long()], torch.sort(codes, stable=True).values)
    assert int(o1[-1]) == codes.numel()
    codes[:10] = 49  # in-place write: a new version, a new index
    p3, o3 = bag_index(codes, 50)
    assert p3 is not p1
    assert torch.equal(codes[p3.long()], torch.sort(codes, stable=True).values)

"""GPU parity of the trainable LLP query (SURVEY config 4 shape, small n)
against golden values from the reference's own train() loop.

Tolerance: rtol 1e-5 for losses, weights and gradients (north-star LLP
tolerance); exact-swap keys and counts bit-exact.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200.storage import tensor_type

pytestmark = pytest.mark.gpu

G = Path(__file__).resolve().parent / "golden"
A = np.load(G / "golden.npz")
META = json.loads((G / "golden.json").read_text())
BAGS = 25


def _setup():
    X, bag, target = A["llp/X"], A["llp/bag"], A["llp/target"]
    model = tq.Linear(X.shape[1], 2, np.random.default_rng(5), name="lin", dtype="float64")
    np.testing.assert_array_equal(model.weight.value.numpy(), A["llp/W0"])
    bag_pe = tq.one_hot_pe(bag, BAGS)
    reg = tq.UdfRegistry()
    reg.register(tq.UdfEntry("llp", (("Bag", tensor_type(BAGS)), ("Pred", tensor_type(2))), 1,
                             lambda c: (bag_pe, tq.pe_encode(model(c.values))), model.parameters))
    cat = tq.Catalog()
    cat.register_tensor(tq.Tensor(X), "T")
    plan = tq.lower(tq.bind(tq.parse("SELECT Bag, Pred, COUNT(*) FROM llp(T) GROUP BY Bag, Pred"),
                            cat, reg))
    q = tq.compile_plan(plan, tq.CompileConfig(trainable=True), reg)
    return X, target, model, cat, q, plan


def test_llp_train_matches_reference():
    X, target, model, cat, q, plan = _setup()
    assert tq.explain(plan) == META["plans"]["llp"]["explain"]
    assert q.explain_compiled() == META["plans"]["llp"]["compiled"]
    assert q.swap_to_exact().explain_compiled() == META["plans"]["llp"]["exact"]
    losses = tq.train(q, cat, [("T", tq.Tensor(X), tq.Tensor(target))],
                      tq.TrainConfig(iterations=4, lr=0.05))
    np.testing.assert_allclose(losses, A["llp/losses"], rtol=1e-5)
    np.testing.assert_allclose(model.weight.value.numpy(), A["llp/W4"], rtol=1e-5, atol=1e-8)
    np.testing.assert_allclose(model.bias.value.numpy(), A["llp/b4"], rtol=1e-5, atol=1e-8)
    res = q.run(cat)
    pred = res.columns[2].values
    loss = tq.mse_loss(pred, tq.Tensor(target))
    tq.backward(loss)
    np.testing.assert_allclose(pred.numpy(), A["llp/grid5"], rtol=1e-5)
    np.testing.assert_allclose(q.tape.gradient(model.weight.value).numpy(), A["llp/dW5"],
                               rtol=1e-5, atol=1e-9)
    np.testing.assert_allclose(q.tape.gradient(model.bias.value).numpy(), A["llp/db5"],
                               rtol=1e-5, atol=1e-9)
    q.end_session()
    exact = q.swap_to_exact().run(cat)
    for nm, col in zip(exact.schema.names, exact.columns):
        np.testing.assert_array_equal(col.values.numpy(), A[f"llp/exact/{nm}"])


def test_soft_counts_conserve_mass_and_gradient_of_total_is_zero():
    rng = np.random.default_rng(3)
    logits = rng.normal(size=(4000, 3))
    with tq.Tape() as tape:
        x = tq.Tensor(logits)
        pe = tq.pe_encode(x)
        c = tq.soft_count(pe)
        from paper_2211_02753_b200.tensor import reduce_sum

        total = reduce_sum(c)
        tq.backward(total)
        g = tape.gradient(x).numpy()
    assert abs(float(total.item()) - 4000.0) < 1e-6
    assert np.max(np.abs(g)) < 1e-6


@pytest.mark.parametrize("dtype,d", [("float64", 32), ("float32", 64)])
def test_exact_swap_fused_argmax_count(dtype, d):
    """swap_to_exact of an LLP-shaped query: COUNT by (decoded one-hot bag,
    argmax of the linear head's softmax) in one pass over X
    (tdp_linear_argmax_count) == decoding the materialised probabilities
    (same row arithmetic) and counting, bit for bit; and == numpy in float64."""
    from paper_2211_02753_b200.encodings import DecodedArgmax

    rng = np.random.default_rng(7)
    n, bags, k = 50_000, 37, 3
    X = rng.normal(size=(n, d)).astype(dtype)
    bag = rng.integers(0, bags, size=n)
    model = tq.Linear(d, k, np.random.default_rng(1), name="lin", dtype=dtype)
    bag_pe = tq.one_hot_pe(bag, bags)
    reg = tq.UdfRegistry()
    reg.register(tq.UdfEntry("llp", (("Bag", tensor_type(bags)), ("Pred", tensor_type(k))), 1,
                             lambda c: (bag_pe, tq.pe_encode(model(c.values))), model.parameters))
    cat = tq.Catalog()
    cat.register_tensor(tq.Tensor(X), "T")
    plan = tq.lower(tq.bind(tq.parse("SELECT Bag, Pred, COUNT(*) FROM llp(T) GROUP BY Bag, Pred"),
                            cat, reg))
    exact = tq.compile_plan(plan, tq.CompileConfig(trainable=True), reg).swap_to_exact()
    dec = tq.pe_decode(tq.pe_encode(model(tq.Tensor(X))))
    assert isinstance(dec.values._lazy, DecodedArgmax)  # the fused path's input form
    res = exact.run(cat)
    got = [c.values.numpy() for c in res.columns]
    # eager: materialise P with the unfused kernels, decode, count
    P = tq.pe_encode(model(tq.Tensor(X))).values.numpy()
    pred = np.argmax(P, axis=1)
    cells, cnt = np.unique(bag * k + pred, return_counts=True)
    np.testing.assert_array_equal(got[0], cells // k)
    np.testing.assert_array_equal(got[1], cells % k)
    np.testing.assert_array_equal(got[2], cnt)
    if dtype == "float64":
        z = X @ model.weight.value.numpy() + model.bias.value.numpy()
        e = np.exp(z - z.max(axis=1, keepdims=True))
        ref = np.argmax(e / e.sum(axis=1, keepdims=True), axis=1)
        assert np.count_nonzero(ref != pred) == 0


@pytest.mark.parametrize("optimizer", ["adam", "sgd"])
def test_graphed_training_equals_eager(optimizer, monkeypatch):
    """tq.train() captures one iteration (query run, MSE, backward, optimizer
    step) in a CUDA graph after two eager ones and replays it: the losses and
    the trained weights equal the all-eager loop's (the one-pass LLP kernel,
    fp32 X, 1000 bags; Adam's bias correction read from a device table)."""
    import torch

    from paper_2211_02753_b200 import training as T

    rng = np.random.default_rng(11)
    n, d, bags = 120_000, 64, 1000
    X = torch.tensor(rng.normal(size=(n, d)), dtype=torch.float32, device="cuda")
    bag = torch.tensor(rng.integers(0, bags, size=n), device="cuda")
    target = torch.tensor(rng.random(bags * 2) * (n / bags / 2), dtype=torch.float64,
                          device="cuda")

    def run(graph: bool):
        monkeypatch.setenv("TDP_TRAIN_GRAPH", "1" if graph else "0")
        model = tq.Linear(d, 2, np.random.default_rng(0), name="lin")
        bag_pe = tq.one_hot_pe(bag, bags)
        reg = tq.UdfRegistry()
        reg.register(tq.UdfEntry("llp", (("Bag", tensor_type(bags)), ("Pred", tensor_type(2))), 1,
                                 lambda c: (bag_pe, tq.pe_encode(model(c.values))),
                                 model.parameters))
        cat = tq.Catalog()
        xt = tq.Tensor(X)
        cat.register_tensor(xt, "T")
        q = tq.compile_plan(tq.lower(tq.bind(tq.parse(
            "SELECT Bag, Pred, COUNT(*) FROM llp(T) GROUP BY Bag, Pred"), cat, reg)),
            tq.CompileConfig(trainable=True), reg)
        losses = tq.train(q, cat, [("T", xt, tq.Tensor(target))],
                          tq.TrainConfig(iterations=7, lr=0.01, optimizer=optimizer))
        return losses, model.weight.value.numpy(), model.bias.value.numpy()

    before = T.GRAPHED[0]
    lg, wg, bg = run(True)
    assert T.GRAPHED[0] == before + 1  # captured once, replayed five times
    le, we, be = run(False)
    assert T.GRAPHED[0] == before + 1
    np.testing.assert_allclose(lg, le, rtol=1e-12)
    np.testing.assert_allclose(wg, we, rtol=1e-12, atol=0)
    np.testing.assert_allclose(bg, be, rtol=1e-12, atol=0)

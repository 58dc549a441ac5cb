"""GPU: differentiable ORDER BY [LIMIT k] for trainable queries (SURVEY §8(f)
4; new semantics -- the reference rejects it, tq/compiler.py:464-475):
the NeuralSort relaxation (csrc/softsort.cu) against a float64 torch
restatement, forward rows and score gradients at rtol 1e-9."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200.autograd import soft_sort_matrix

pytestmark = pytest.mark.gpu


def _neuralsort(s: torch.Tensor, k: int, tau: float) -> torch.Tensor:
    n = s.numel()
    B = (s[:, None] - s[None, :]).abs().sum(dim=1)
    c = (n + 1 - 2 * torch.arange(1, k + 1, dtype=s.dtype, device=s.device))
    return torch.softmax((c[:, None] * s[None, :] - B[None, :]) / tau, dim=1)


@pytest.mark.parametrize("n,k,tau", [(7, 7, 1.0), (300, 10, 0.5), (5000, 64, 2.0), (1000, 1000, 0.1)])
def test_soft_sort_rows_and_gradient_match_float64(n, k, tau):
    g = torch.Generator(device="cuda").manual_seed(n)
    s = torch.randn(n, generator=g, device="cuda", dtype=torch.float64) * 3
    s[: n // 10] = s[0]  # ties
    W = torch.randn((k, n), generator=g, device="cuda", dtype=torch.float64)
    a = s.clone().requires_grad_(True)
    P = soft_sort_matrix(a, k, tau)
    (P * W).sum().backward()
    b = s.clone().requires_grad_(True)
    R = _neuralsort(b, k, tau)
    (R * W).sum().backward()
    torch.testing.assert_close(P, R, rtol=1e-9, atol=1e-12)
    torch.testing.assert_close(a.grad, b.grad, rtol=1e-8, atol=1e-10)


def test_soft_sort_tends_to_the_hard_order():
    g = torch.Generator(device="cuda").manual_seed(1)
    s = torch.randn(200, generator=g, device="cuda", dtype=torch.float64)
    P = soft_sort_matrix(s, 20, 1e-4)
    order = torch.argsort(s, descending=True)[:20]
    assert torch.equal(P.argmax(dim=1), order)
    assert float((P.max(dim=1).values - 1).abs().max()) < 1e-9


def _query(X, tau, limit, desc=True):
    from paper_2211_02753_b200.storage import FLOAT, INT
    from paper_2211_02753_b200.tensor import reshape

    n, d = X.shape
    lin = tq.Linear(d, 1, np.random.default_rng(3), name="sc", dtype="float64")
    ids = tq.Tensor(np.arange(n, dtype=np.int64))
    reg = tq.UdfRegistry()
    reg.register(tq.UdfEntry("sc", (("id", INT), ("s", FLOAT)), 1,
                             lambda c: (tq.plain(ids), tq.plain(reshape(lin(c.values), (n,)))),
                             lin.parameters, pe_outputs=False))
    cat = tq.Catalog()
    cat.register_tensor(tq.Tensor(X), "T")
    sql = f"SELECT id, s FROM sc(T) ORDER BY s {'DESC' if desc else ''} LIMIT {limit}"
    q = tq.compile_plan(tq.lower(tq.bind(tq.parse(sql), cat, reg)),
                        tq.CompileConfig(trainable=True, soft_sort_tau=tau), reg)
    return q, cat, lin


@pytest.mark.parametrize("desc", [True, False])
def test_trainable_order_by_limit_query(desc):
    """SELECT id, s FROM sc(T) ORDER BY s [DESC] LIMIT 8, trainable: the id
    column is the exact stable order, the score column the relaxed top-8;
    parameter gradients of an MSE on the soft scores equal float64 torch."""
    from paper_2211_02753_b200.tensor import backward
    from paper_2211_02753_b200.training import mse_loss

    rng = np.random.default_rng(11)
    X = rng.normal(size=(500, 6))
    tau, k = 0.7, 8
    q, cat, lin = _query(X, tau, k, desc)
    assert "sort[soft]" in q.explain_compiled()
    res = q.run(cat)
    target = tq.Tensor(np.linspace(3.0, 1.0, k))
    loss = mse_loss(res.columns[1].values, target)
    backward(loss)
    dW = q.tape.gradient(lin.weight.value).numpy()
    db = q.tape.gradient(lin.bias.value).numpy()
    ids = res.columns[0].values.numpy()
    q.end_session()
    # float64 torch restatement
    W = torch.tensor(lin.weight.value.numpy(), device="cuda", requires_grad=True)
    b = torch.tensor(lin.bias.value.numpy(), device="cuda", requires_grad=True)
    Xt = torch.tensor(X, device="cuda")
    s = (Xt @ W + b).reshape(-1)
    P = _neuralsort(s if desc else -s, k, tau)
    soft = P @ s
    ref_loss = ((soft - torch.tensor(np.linspace(3.0, 1.0, k), device="cuda")) ** 2).mean()
    ref_loss.backward()
    np.testing.assert_allclose(res.columns[1].values.numpy(), soft.detach().cpu().numpy(),
                               rtol=1e-9)
    np.testing.assert_allclose(dW, W.grad.cpu().numpy(), rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(db, b.grad.cpu().numpy(), rtol=1e-8, atol=1e-12)
    sv = s.detach().cpu().numpy()
    exp_ids = np.argsort(-sv if desc else sv, kind="stable")[:k]
    np.testing.assert_array_equal(ids, exp_ids)


def test_trainable_order_by_learns_a_ranking():
    """tq.train on a soft top-k: the loss falls."""
    rng = np.random.default_rng(2)
    X = rng.normal(size=(400, 6))
    q, cat, lin = _query(X, 0.5, 5)
    losses = tq.train(q, cat, [("T", tq.Tensor(X), tq.Tensor(np.full(5, 4.0)))],
                      tq.TrainConfig(iterations=30, lr=0.05))
    assert losses[-1] < 0.5 * losses[0]

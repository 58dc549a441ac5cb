"""GPU: image query with a CNN UDF (SURVEY config 5 shape, small n).

The reference has no convolution op, so the check is against a plain PyTorch
float64 CPU computation of the same query (softmax -> column sums -> MSE) and
its autograd gradients; rtol 1e-5.  The exact swap's counts must equal the
argmax histogram bit-exactly.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200.models import TorchModel

pytestmark = pytest.mark.gpu


def _cnn(k: int) -> torch.nn.Module:
    torch.manual_seed(0)
    return torch.nn.Sequential(
        torch.nn.Unflatten(1, (1, 28)),
        torch.nn.Conv2d(1, 8, 3), torch.nn.ReLU(), torch.nn.MaxPool2d(2),
        torch.nn.Conv2d(8, 16, 3), torch.nn.ReLU(), torch.nn.MaxPool2d(2),
        torch.nn.Flatten(), torch.nn.Linear(400, k))


@pytest.mark.parametrize("chunk_rows", [0, 128])
def test_cnn_image_query_matches_torch_reference(chunk_rows):
    k, n = 4, 600
    rng = np.random.default_rng(0)
    images = rng.random((n, 28, 28)).astype(np.float64)
    target = np.array([150.0, 150.0, 200.0, 100.0])
    net = _cnn(k).double()
    ref_net = _cnn(k).double()
    ref_net.load_state_dict(net.state_dict())
    net = net.cuda()
    model = TorchModel(net, "cnn", chunk_rows=chunk_rows)
    reg = tq.UdfRegistry()
    reg.register(tq.classifier_tvf("cnn", model, k, "Pred"))
    cat = tq.Catalog()
    cat.register_tensor(tq.Tensor(images), "imgs")
    plan = tq.lower(tq.bind(tq.parse("SELECT Pred, COUNT(*) FROM cnn(imgs) GROUP BY Pred"), cat, reg))
    q = tq.compile_plan(plan, tq.CompileConfig(trainable=True), reg)
    assert [p.name for p in q.parameters()][:2] == ["cnn.1.weight", "cnn.1.bias"]

    res = q.run(cat)
    pred = res.columns[1].values
    loss = tq.mse_loss(pred, tq.Tensor(target))
    tq.backward(loss)
    grads = [q.tape.gradient(p.value).numpy() for p in q.parameters()]
    q.end_session()

    x = torch.from_numpy(images)
    counts = torch.softmax(ref_net(x), dim=1).sum(dim=0)
    ref_loss = torch.mean((counts - torch.from_numpy(target)) ** 2)
    ref_loss.backward()
    np.testing.assert_allclose(pred.numpy(), counts.detach().numpy(), rtol=1e-5)
    np.testing.assert_allclose(float(loss.item()), float(ref_loss.detach()), rtol=1e-5)
    for g, p in zip(grads, ref_net.parameters()):
        np.testing.assert_allclose(g, p.grad.numpy(), rtol=1e-5, atol=1e-9)

    exact = q.swap_to_exact().run(cat)
    labels = torch.argmax(ref_net(x), dim=1).numpy()
    keys, cnts = np.unique(labels, return_counts=True)
    np.testing.assert_array_equal(exact.columns[0].values.numpy(), keys)
    np.testing.assert_array_equal(exact.columns[1].values.numpy(), cnts)


def test_cnn_query_trains():
    k, n = 3, 400
    rng = np.random.default_rng(1)
    images = rng.random((n, 28, 28)).astype(np.float32)
    net = _cnn(k).cuda()
    model = TorchModel(net, "cnn")
    reg = tq.UdfRegistry()
    reg.register(tq.classifier_tvf("cnn", model, k, "Pred"))
    cat = tq.Catalog()
    plan_sql = "SELECT Pred, COUNT(*) FROM cnn(imgs) GROUP BY Pred"
    cat.register_tensor(tq.Tensor(images), "imgs")
    q = tq.compile_plan(tq.lower(tq.bind(tq.parse(plan_sql), cat, reg)),
                        tq.CompileConfig(trainable=True), reg)
    target = tq.Tensor(np.array([300.0, 50.0, 50.0], dtype=np.float32))
    losses = tq.train(q, cat, [("imgs", tq.Tensor(images), target)],
                      tq.TrainConfig(iterations=30, lr=0.01))
    assert losses[-1] < 0.5 * losses[0]

"""Trainable (soft) query cases shared by make_soft_golden.py (runs the
reference) and tests/test_gpu_soft_golden.py (runs this package): the data,
the models and the UDFs are built the same way for either implementation
(`api`: the reference package or this one)."""

from __future__ import annotations

from importlib import import_module

import numpy as np

BAGS = 7


def data(n: int, d: int, seed: int) -> dict[str, np.ndarray]:
    rng = np.random.default_rng(seed)
    return {"X": rng.normal(size=(n, d)), "bag": rng.integers(0, BAGS, size=n).astype(np.int64),
            "v": np.round(rng.normal(size=n) * 3, 2)}


def build(api, d_arr: dict, k: int, k2: int, seed: int):
    """(catalog, registry, models): table T (the feature rows), and UDFs
    clf(T) -> Pred [k] | pair(T) -> (Bag one-hot [BAGS], Pred [k]) |
    two(T) -> (P1 [k], P2 [k2]) | val(T) -> (Pred [k], val float)."""
    storage = import_module(api.__name__ + ".storage")
    tensor = import_module(api.__name__ + ".tensor")
    X, bag, v = d_arr["X"], d_arr["bag"], d_arr["v"]
    n, d = X.shape
    lin = api.Linear(d, k, np.random.default_rng(seed), name="lin", dtype="float64")
    lin2 = api.Linear(d, k2, np.random.default_rng(seed + 1), name="lin2", dtype="float64")
    bag_pe = api.one_hot_pe(bag, BAGS)
    vcol = api.plain(api.Tensor(v))
    reg = api.UdfRegistry()
    T = storage.tensor_type
    reg.register(api.UdfEntry("clf", (("Pred", T(k)),), 1,
                              lambda c: (api.pe_encode(lin(c.values)),), lin.parameters))
    reg.register(api.UdfEntry("pair", (("Bag", T(BAGS)), ("Pred", T(k))), 1,
                              lambda c: (bag_pe, api.pe_encode(lin(c.values))), lin.parameters))
    reg.register(api.UdfEntry("two", (("P1", T(k)), ("P2", T(k2))), 1,
                              lambda c: (api.pe_encode(lin(c.values)),
                                         api.pe_encode(lin2(c.values))),
                              lin.parameters + lin2.parameters))
    reg.register(api.UdfEntry("val", (("Pred", T(k)), ("val", storage.FLOAT)), 1,
                              lambda c: (api.pe_encode(lin(c.values)), vcol), lin.parameters))

    def score(c):
        s = tensor.reshape(lin2(c.values), (c.values.shape[0],)) if k2 == 1 else None
        return (api.plain(s),)

    if k2 == 1:
        reg.register(api.UdfEntry("sc", (("s", storage.FLOAT),), 1, score, lin2.parameters,
                                  pe_outputs=False))
    cat = api.Catalog()
    cat.register_tensor(api.Tensor(X), "T")
    return cat, reg, (lin, lin2)


QUERIES = [
    "SELECT Pred, COUNT(*) FROM clf(T) GROUP BY Pred",
    "SELECT Bag, Pred, COUNT(*) FROM pair(T) GROUP BY Bag, Pred",
    "SELECT Pred, Bag, COUNT(*) FROM pair(T) GROUP BY Pred, Bag",
    "SELECT P1, P2, COUNT(*) FROM two(T) GROUP BY P1, P2",
    "SELECT Pred, SUM(val), AVG(val), COUNT(*) FROM val(T) GROUP BY Pred",
    "SELECT Pred, AVG(val) FROM val(T) GROUP BY Pred",
    "SELECT SUM(s), AVG(s), COUNT(*) FROM sc(T)",
    "SELECT SUM(s), COUNT(*) FROM (SELECT s FROM sc(T) WHERE s > 0.1)",
]

# (n rows, d features, k classes, k2 classes of the second head / 1: the score
# head of `sc`, seed); a query that needs a head the shape lacks is skipped
SHAPES = [(300, 5, 3, 1, 11), (2000, 8, 2, 4, 12), (1500, 4, 4, 1, 13), (64, 3, 5, 2, 14)]


def applicable(sql: str, k2: int) -> bool:
    if "sc(T)" in sql:
        return k2 == 1
    if "two(T)" in sql:
        return k2 >= 2
    return True


def run_case(api, sql: str, shape, tape_grad):
    """Run one trainable query; loss = sum_j sum(G_j * float column j) with
    seeded weights G; returns (names, outputs, {param name: gradient})."""
    tensor = import_module(api.__name__ + ".tensor")
    n, d, k, k2, seed = shape
    cat, reg, models = build(api, data(n, d, seed), k, k2, seed)
    plan = api.lower(api.bind(api.parse(sql), cat, reg))
    q = api.compile_plan(plan, api.CompileConfig(trainable=True), reg)
    res = q.run(cat)
    names = list(res.schema.names)
    rng = np.random.default_rng(seed + 100)
    loss = tensor.tensor(0.0)
    outs = []
    for col in res.columns:
        vals = col.values
        outs.append(np.asarray(vals.numpy() if hasattr(vals, "numpy") else vals.data))
        if outs[-1].dtype.kind == "f":
            g = rng.normal(size=outs[-1].shape)
            loss = tensor.add(loss, tensor.reduce_sum(tensor.mul(vals, tensor.tensor(g))))
    tensor.backward(loss)
    grads = {}
    for m in models:
        for p in m.parameters:
            g = q.tape.gradient(p.value)
            if g is not None:
                grads[p.name] = tape_grad(g)
    q.end_session()
    return names, outs, grads

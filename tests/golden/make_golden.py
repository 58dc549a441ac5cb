"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (the reference is importable there, not on the
GPU host):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz (arrays) and tests/golden/golden.json (plan
dumps, metadata).  Every case records its inputs and the reference's outputs;
tests/test_oracle_golden.py pins the oracle to them and
tests/test_gpu_golden.py checks the B200 path against them.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

import tensorquery as ref  # noqa: E402
from tensorquery import kernels as rk  # noqa: E402
from tensorquery import compiler as rc  # noqa: E402
from tensorquery.encodings import (  # noqa: E402
    DictionaryEncoding, EncodedTensor, ProbabilityEncoding, StringDictionary, plain)
from tensorquery.tensor import Tape, Tensor, backward, mul, reduce_sum, tensor  # noqa: E402

from paper_2211_02753_b200 import workloads as wl  # noqa: E402  (generators only)

arrays: dict[str, np.ndarray] = {}
meta: dict = {}


def put(name, value):
    arrays[name] = np.asarray(value)


# ---------------------------------------------------------------------------
# filter cases (comparison_mask semantics incl. NEP 50 literal promotion)
# ---------------------------------------------------------------------------
rng = np.random.default_rng(1234)
n = 257
cols = {
    "i64": rng.integers(-20, 20, size=n).astype(np.int64),
    "f64": np.round(rng.normal(size=n), 2),
    "f32": (rng.integers(0, 11, size=n) / 100).astype(np.float32),
    "big": rng.integers(2**53 - 4, 2**53 + 4, size=n).astype(np.int64),
}
cols["f64"][:3] = [np.nan, -0.0, np.inf]
filter_cases = [
    [("i64", ">=", 3), ("f64", "<", 0.5)],
    [("f32", "<=", 0.07), ("f32", ">=", 0.05)],
    [("i64", "<", 2.5)],
    [("i64", "<>", 0)],
    [("big", ">", 2.0**53)],
    [("big", "=", 2**53 + 1)],
    [("i64", "<", 2**70)],
    [("i64", ">", -(2**70))],
    [("f64", "=", -0.0)],
    [("f64", "<>", 1.0)],
    [],
]
names = list(cols)
for name, c in cols.items():
    put(f"filter/col/{name}", c)
meta["filter_cases"] = []
for ci, preds in enumerate(filter_cases):
    ets = [plain(Tensor(cols[k])) for k in names]
    p = [(names.index(c), op, lit) for c, op, lit in preds]
    out = rk.filter_exact(ets, p)
    meta["filter_cases"].append([[c, op, lit] for c, op, lit in preds])
    for k, o in zip(names, out):
        put(f"filter/{ci}/{k}", o.values.data)

# dictionary filter incl. absent literal
d = ref.dict_encode(["b", "a", "c", "b", "a", "d"])
put("dictfilter/codes", d.values.data)
meta["dictfilter"] = {"entries": list(d.encoding.dictionary.entries), "cases": []}
for ci, (op, lit) in enumerate([("=", "b"), ("<", "c"), (">", "zz"), ("<>", "a"), ("<", "bb")]):
    out = rk.filter_exact([d], [(0, op, lit)])
    meta["dictfilter"]["cases"].append([op, lit])
    put(f"dictfilter/{ci}", out[0].values.data)

# ---------------------------------------------------------------------------
# exact group-by
# ---------------------------------------------------------------------------
m = 3000
k1 = rng.integers(-3, 4, size=m).astype(np.int64)
k2 = rng.choice(np.array([10**12, -5, 7, 99], dtype=np.int64), size=m)
vf = rng.normal(size=m)
vf32 = rng.normal(size=m).astype(np.float32)
vi = rng.integers(-(2**40), 2**40, size=m).astype(np.int64)
for k, v in {"k1": k1, "k2": k2, "vf": vf, "vf32": vf32, "vi": vi}.items():
    put(f"groupby/in/{k}", v)
keys, aggs = rk.groupby_exact([plain(Tensor(k1)), plain(Tensor(k2))],
                              [("count", None), ("sum", vf), ("avg", vf), ("sum", vf32),
                               ("avg", vf32), ("sum", vi), ("avg", vi)])
for j, kv in enumerate(keys):
    put(f"groupby/out/key{j}", kv)
for j, a in enumerate(aggs):
    put(f"groupby/out/agg{j}", a)
# SPEC example
keys, aggs = rk.groupby_exact([plain(Tensor(np.array([1, 1, 2]))), plain(Tensor(np.array([0, 1, 0])))],
                              [("count", None)])
put("spec/groupby/keys", np.stack(keys))
put("spec/groupby/counts", aggs[0])

# global aggregates
rel = rc.Relation(("vf", "vf32", "vi"), (plain(Tensor(vf)), plain(Tensor(vf32)), plain(Tensor(vi))))
g = rc._global_aggregate(rel, [("count", None), ("sum", vf), ("avg", vf), ("sum", vf32),
                              ("avg", vf32), ("sum", vi), ("avg", vi)])
for j, a in enumerate(g):
    put(f"global/out/{j}", a)
empty = rc._global_aggregate(rc.Relation(("x",), (plain(Tensor(vf[:0])),)),
                             [("count", None), ("sum", vf[:0]), ("avg", vf[:0])])
for j, a in enumerate(empty):
    put(f"global/empty/{j}", a)

# ---------------------------------------------------------------------------
# sort
# ---------------------------------------------------------------------------
si = rng.integers(-5, 5, size=500).astype(np.int64)
si[:2] = [np.iinfo(np.int64).min, np.iinfo(np.int64).max]
sf = (rng.integers(-5, 5, size=500) / 2).astype(np.float64)
sf[:4] = [np.nan, -0.0, 0.0, -np.inf]
put("sort/in/i64", si)
put("sort/in/f64", sf)
for nm, key in (("i64", si), ("f64", sf)):
    for desc in (False, True):
        put(f"sort/out/{nm}/{int(desc)}", rk.stable_order(plain(Tensor(key)), desc))
put("spec/sort_limit", rk.sort_limit([plain(Tensor(np.array([0.2, 0.9, 0.5]))),
                                      plain(Tensor(np.arange(3)))], 0, True, 2)[1].values.data)
put("spec/desc_ties", rk.stable_order(plain(Tensor(np.array([1, 0, 1, 0]))), True))

# ---------------------------------------------------------------------------
# soft path: softmax, pe_decode, soft_groupby forward + reference-tape gradients
# ---------------------------------------------------------------------------
logits = rng.normal(size=(64, 5))
logits[0] = 0.0
put("soft/logits", logits)
with Tape() as tape:
    x = tensor(logits)
    pe = ref.pe_encode(x)
    gsm = rng.normal(size=(64, 5))
    backward(reduce_sum(mul(pe.values, tensor(gsm))))
    put("soft/softmax", pe.values.data)
    put("soft/softmax_grad_in", gsm)
    put("soft/softmax_grad", tape.gradient(x).data)
put("soft/pe_decode", ref.pe_decode(pe).values.data)

p1 = rng.dirichlet(np.ones(3), size=200)
p2 = rng.dirichlet(np.ones(4), size=200)
w = rng.normal(size=200)
G = rng.normal(size=(3, 4))
put("soft/p1", p1)
put("soft/p2", p2)
put("soft/w", w)
put("soft/G", G)
for agg in ("count", "sum", "avg"):
    with Tape() as tape:
        a, b, v = tensor(p1), tensor(p2), tensor(w)
        res = rk.soft_groupby([EncodedTensor(a, ProbabilityEncoding(3)),
                               EncodedTensor(b, ProbabilityEncoding(4))], agg,
                              v if agg != "count" else None)
        backward(reduce_sum(mul(res.counts, tensor(G))))
        put(f"soft/{agg}/grid", res.counts.data)
        put(f"soft/{agg}/dp1", tape.gradient(a).data)
        put(f"soft/{agg}/dp2", tape.gradient(b).data)
        if agg != "count":
            put(f"soft/{agg}/dw", tape.gradient(v).data)

codes = rng.integers(0, 6, size=200)
put("soft/onehot_codes", codes)
with Tape() as tape:
    pb = tensor(p2)
    res = rk.soft_groupby([ref.one_hot_pe(codes, 6), EncodedTensor(pb, ProbabilityEncoding(4))])
    G2 = rng.normal(size=(6, 4))
    backward(reduce_sum(mul(res.counts, tensor(G2))))
    put("soft/onehot/G", G2)
    put("soft/onehot/grid", res.counts.data)
    put("soft/onehot/dp", tape.gradient(pb).data)
put("spec/soft_count", rk.soft_count(EncodedTensor(tensor([[0.9, 0.1], [0.2, 0.8], [0.7, 0.3]]),
                                                   ProbabilityEncoding(2))).data)
put("spec/dense_exact_counts", rk.dense_exact_counts([np.array([0, 1, 1, 2]), np.array([1, 0, 1, 1])],
                                                     [3, 2]))

# ---------------------------------------------------------------------------
# end-to-end Q1 / Q6 through the reference's own SQL -> compile -> run
# ---------------------------------------------------------------------------
li = wl.lineitem_arrays(0.01, seed=99, rows=20_000)
for k, v in li.items():
    put(f"tpch/in/{k}", v)


def ref_catalog():
    cat = ref.Catalog()
    cols = []
    for name in wl.LINEITEM_COLUMNS:
        v = Tensor(li[name])
        if name == "l_returnflag":
            cols.append(EncodedTensor(v, DictionaryEncoding(StringDictionary(("A", "N", "R")))))
        elif name == "l_linestatus":
            cols.append(EncodedTensor(v, DictionaryEncoding(StringDictionary(("F", "O")))))
        else:
            cols.append(plain(v))
    cat.register("lineitem", ref.table_from_columns(list(wl.LINEITEM_COLUMNS), cols))
    return cat


def ref_q1_registry():
    from tensorquery.tensor import add, sub
    from tensorquery.storage import FLOAT, STRING

    def q1prep(rf, ls, q, p, d, t):
        one = tensor(1.0)
        dp = mul(p.values, sub(one, d.values))
        ch = mul(dp, add(one, t.values))
        return (rf, ls, q, p, plain(dp), plain(ch), d)

    reg = ref.UdfRegistry()
    reg.register(ref.UdfEntry("q1prep", (("rf", STRING), ("ls", STRING), ("qty", FLOAT),
                                         ("price", FLOAT), ("disc_price", FLOAT),
                                         ("charge", FLOAT), ("disc", FLOAT)), 6, q1prep, (),
                              pe_outputs=False))
    return reg


def ref_q6_registry():
    from tensorquery.storage import FLOAT

    reg = ref.UdfRegistry()
    reg.register(ref.UdfEntry("revenue", (("rev", FLOAT),), 2,
                              lambda p, d: (plain(mul(p.values, d.values)),), (), pe_outputs=False))
    return reg


meta["plans"] = {}
for qname, sql, reg in (("q1", wl.Q1_SQL, ref_q1_registry()), ("q6", wl.Q6_SQL, ref_q6_registry())):
    cat = ref_catalog()
    plan = ref.lower(ref.bind(ref.parse(sql), cat, reg))
    q = ref.compile_plan(plan, ref.CompileConfig(), reg)
    out = q.run(cat)
    meta["plans"][qname] = {"explain": ref.explain(plan), "compiled": q.explain_compiled(),
                            "names": list(out.schema.names), "to_sql": ref.to_sql(ref.parse(sql))}
    for nm, col in zip(out.schema.names, out.columns):
        put(f"tpch/{qname}/{nm}", col.values.data)

# ---------------------------------------------------------------------------
# LLP: trainable soft group-by-count through the reference's own train()
# (SURVEY Appendix A llp TVF; float64 model for parity)
# ---------------------------------------------------------------------------
from tensorquery.storage import tensor_type  # noqa: E402

llp_rng = np.random.default_rng(77)
n_llp, d_llp, bags = 3000, 8, 25
X = llp_rng.normal(size=(n_llp, d_llp))
bag = llp_rng.integers(0, bags, size=n_llp)
Wstar = llp_rng.normal(size=(d_llp, 2))
labels = np.argmax(X @ Wstar, axis=1)
target = np.zeros((bags, 2))
np.add.at(target, (bag, labels), 1.0)
put("llp/X", X)
put("llp/bag", bag)
put("llp/target", target.reshape(-1))
model = ref.Linear(d_llp, 2, np.random.default_rng(5), name="lin", dtype="float64")
put("llp/W0", model.weight.value.data.copy())
reg = ref.UdfRegistry()
reg.register(ref.UdfEntry("llp", (("Bag", tensor_type(bags)), ("Pred", tensor_type(2))), 1,
                          lambda c: (ref.one_hot_pe(bag, bags), ref.pe_encode(model(c.values))),
                          model.parameters))
cat = ref.Catalog()
cat.register_tensor(Tensor(X), "T")
sql = "SELECT Bag, Pred, COUNT(*) FROM llp(T) GROUP BY Bag, Pred"
plan = ref.lower(ref.bind(ref.parse(sql), cat, reg))
q = ref.compile_plan(plan, ref.CompileConfig(trainable=True), reg)
meta["plans"]["llp"] = {"explain": ref.explain(plan), "compiled": q.explain_compiled(),
                        "exact": q.swap_to_exact().explain_compiled()}
losses = ref.train(q, cat, [("T", Tensor(X), Tensor(target.reshape(-1)))],
                   ref.TrainConfig(iterations=4, lr=0.05))
put("llp/losses", np.array(losses))
put("llp/W4", model.weight.value.data.copy())
put("llp/b4", model.bias.value.data.copy())
# one more forward + gradient at the trained weights
res = q.run(cat)
pred = res.columns[2].values
loss = ref.mse_loss(pred, Tensor(target.reshape(-1)))
backward(loss)
put("llp/grid5", pred.data)
put("llp/dW5", q.tape.gradient(model.weight.value).data)
put("llp/db5", q.tape.gradient(model.bias.value).data)
q.end_session()
exact = q.swap_to_exact().run(cat)
for nm, col in zip(exact.schema.names, exact.columns):
    put(f"llp/exact/{nm}", col.values.data)

# ---------------------------------------------------------------------------
# gradient paths through gather (take_rows' VJP, tq/tensor.py:597-614) and the
# trainable global aggregates (GlobalAggSoftOp, tq/compiler.py:265-288)
# ---------------------------------------------------------------------------
from tensorquery.tensor import gather  # noqa: E402

g_rng = np.random.default_rng(31)
src = g_rng.normal(size=(50, 3))
idx = g_rng.integers(0, 50, size=200)  # duplicates: np.add.at accumulates
gw = g_rng.normal(size=(200, 3))
put("gather/src", src)
put("gather/idx", idx)
put("gather/w", gw)
with Tape() as tape:
    a = Tensor(src)
    out = gather(a, Tensor(idx.astype(np.int64)), axis=0)
    backward(reduce_sum(mul(out, tensor(gw))))
    put("gather/out", out.data)
    put("gather/grad", tape.gradient(a).data)

# trainable query: Linear(6,1) score UDF -> WHERE score > 0.05 (filter_exact ->
# take_rows -> gather on the tape) -> SUM / AVG / COUNT (GlobalAggSoftOp)
n_t, d_t = 400, 6
Xt = g_rng.normal(size=(n_t, d_t))
put("globsoft/X", Xt)
lin = ref.Linear(d_t, 1, np.random.default_rng(8), name="sc", dtype="float64")
put("globsoft/W", lin.weight.value.data.copy())
put("globsoft/b", lin.bias.value.data.copy())
from tensorquery.storage import FLOAT  # noqa: E402
from tensorquery.tensor import reshape as t_reshape  # noqa: E402

regs = ref.UdfRegistry()
regs.register(ref.UdfEntry(
    "sc", (("s", FLOAT),), 1,
    lambda c: (plain(t_reshape(lin(c.values), (c.values.shape[0],))),),
    lin.parameters, pe_outputs=False))
cat = ref.Catalog()
cat.register_tensor(Tensor(Xt), "T")
meta["globsoft"] = {}
for tag, sql in (("filtered", "SELECT SUM(s), AVG(s), COUNT(*) FROM (SELECT s FROM sc(T) "
                              "WHERE s > 0.05)"),
                 ("plain", "SELECT SUM(s), AVG(s), COUNT(*) FROM sc(T)")):
    plan = ref.lower(ref.bind(ref.parse(sql), cat, regs))
    q = ref.compile_plan(plan, ref.CompileConfig(trainable=True), regs)
    meta["globsoft"][tag] = {"sql": sql, "compiled": q.explain_compiled()}
    res = q.run(cat)
    gvec = g_rng.normal(size=2)
    put(f"globsoft/{tag}/G", gvec)
    loss = ref.tensor(0.0)
    from tensorquery.tensor import add as t_add  # noqa: E402

    for j, col in enumerate(res.columns[:2]):
        loss = t_add(loss, reduce_sum(mul(col.values, tensor(gvec[j:j + 1]))))
    backward(loss)
    for nm, col in zip(res.schema.names, res.columns):
        put(f"globsoft/{tag}/{nm}", col.values.data)
    put(f"globsoft/{tag}/dW", q.tape.gradient(lin.weight.value).data)
    put(f"globsoft/{tag}/db", q.tape.gradient(lin.bias.value).data)
    meta["globsoft"][tag]["names"] = list(res.schema.names)
    q.end_session()

np.savez_compressed(HERE / "golden.npz", **arrays)
(HERE / "golden.json").write_text(json.dumps(meta, indent=1, default=float))
print(f"wrote {len(arrays)} arrays")

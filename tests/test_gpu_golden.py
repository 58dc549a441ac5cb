"""GPU: the B200 path against golden vectors produced by the REFERENCE itself
(tests/golden/make_golden.py).  Bit-exact for rows / keys / counts / integer
sums / orders and output dtypes; float aggregates rtol 1e-9 (float64
accumulation in both, different order); soft path rtol 1e-9 (fixed-point count
grid: atol n * 2^-31)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200 import compiler as C
from paper_2211_02753_b200 import kernels as K
from paper_2211_02753_b200.encodings import DictionaryEncoding, StringDictionary
from paper_2211_02753_b200.tensor import Tape, backward, mul, reduce_sum

pytestmark = pytest.mark.gpu

G = Path(__file__).resolve().parent / "golden"
A = np.load(G / "golden.npz")
META = json.loads((G / "golden.json").read_text())


def _col(x):
    return tq.plain(tq.Tensor(x))


def test_filter_cases():
    names = ["i64", "f64", "f32", "big"]
    cols = [_col(A[f"filter/col/{k}"]) for k in names]
    for ci, preds in enumerate(META["filter_cases"]):
        p = [(names.index(c), op, lit) for c, op, lit in preds]
        out = K.filter_exact(cols, p)
        for k, o in zip(names, out):
            got = o.values.numpy()
            exp = A[f"filter/{ci}/{k}"]
            assert got.dtype == exp.dtype
            np.testing.assert_array_equal(got, exp, err_msg=f"case {ci} {preds}")


def test_comparison_mask_matches_filter_rows():
    names = ["i64", "f64", "f32", "big"]
    for ci, preds in enumerate(META["filter_cases"]):
        if len(preds) != 1:
            continue
        c, op, lit = preds[0]
        col = _col(A[f"filter/col/{c}"])
        m = K.comparison_mask(col, op, lit).cpu().numpy()
        np.testing.assert_array_equal(A[f"filter/col/{c}"][m], A[f"filter/{ci}/{c}"])


def test_dictionary_filter_cases():
    entries = tuple(META["dictfilter"]["entries"])
    col = tq.EncodedTensor(tq.Tensor(A["dictfilter/codes"]), DictionaryEncoding(StringDictionary(entries)))
    for ci, (op, lit) in enumerate(META["dictfilter"]["cases"]):
        out = K.filter_exact([col], [(0, op, lit)])
        np.testing.assert_array_equal(out[0].values.numpy(), A[f"dictfilter/{ci}"])
        assert out[0].encoding == col.encoding


def test_groupby_and_global_aggregates():
    k1, k2 = A["groupby/in/k1"], A["groupby/in/k2"]
    vf, vf32, vi = A["groupby/in/vf"], A["groupby/in/vf32"], A["groupby/in/vi"]
    aggs = [("count", None), ("sum", tq.Tensor(vf)), ("avg", tq.Tensor(vf)),
            ("sum", tq.Tensor(vf32)), ("avg", tq.Tensor(vf32)), ("sum", tq.Tensor(vi)),
            ("avg", tq.Tensor(vi))]
    keys, out = K.groupby_exact([_col(k1), _col(k2)], aggs)
    for j, kv in enumerate(keys):
        np.testing.assert_array_equal(kv.cpu().numpy(), A[f"groupby/out/key{j}"])
    for j, o in enumerate(out):
        got, exp = o.cpu().numpy(), A[f"groupby/out/agg{j}"]
        assert got.dtype == exp.dtype, (j, got.dtype, exp.dtype)
        if exp.dtype.kind == "f":
            np.testing.assert_allclose(got, exp, rtol=1e-9)
        else:
            np.testing.assert_array_equal(got, exp)
    rel = C.Relation(("vf", "vf32", "vi"), (_col(vf), _col(vf32), _col(vi)))
    g = C._global_aggregate(rel, aggs)
    for j, o in enumerate(g):
        got, exp = o.cpu().numpy(), A[f"global/out/{j}"]
        assert got.dtype == exp.dtype, (j, got.dtype, exp.dtype)
        np.testing.assert_allclose(got, exp, rtol=1e-6 if exp.dtype == np.float32 else 1e-9)
    empty = C._global_aggregate(C.Relation(("x",), (_col(vf[:0]),)),
                                [("count", None), ("sum", tq.Tensor(vf[:0])), ("avg", tq.Tensor(vf[:0]))])
    for j, o in enumerate(empty):
        got, exp = o.cpu().numpy(), A[f"global/empty/{j}"]
        assert got.dtype == exp.dtype
        np.testing.assert_array_equal(got, exp)


def test_spec_examples():
    keys, aggs = K.groupby_exact([_col(np.array([1, 1, 2])), _col(np.array([0, 1, 0]))],
                                 [("count", None)])
    np.testing.assert_array_equal(np.stack([k.cpu().numpy() for k in keys]), A["spec/groupby/keys"])
    np.testing.assert_array_equal(aggs[0].cpu().numpy(), A["spec/groupby/counts"])
    out = K.sort_limit([_col(np.array([0.2, 0.9, 0.5])), _col(np.arange(3))], 0, True, 2)
    np.testing.assert_array_equal(out[1].values.numpy(), A["spec/sort_limit"])
    np.testing.assert_array_equal(K.stable_order(_col(np.array([1, 0, 1, 0])), True).cpu().numpy(),
                                  A["spec/desc_ties"])
    dec = tq.pe_decode(tq.EncodedTensor(tq.tensor([[0.5, 0.5]]), tq.ProbabilityEncoding(2)))
    assert dec.values.tolist() == [0]
    np.testing.assert_array_equal(
        K.dense_exact_counts([np.array([0, 1, 1, 2]), np.array([1, 0, 1, 1])], [3, 2]).cpu().numpy(),
        A["spec/dense_exact_counts"])
    d = tq.dict_encode(["b", "a", "b"])
    assert d.values.tolist() == [1, 0, 1]


@pytest.mark.parametrize("name", ["i64", "f64"])
@pytest.mark.parametrize("desc", [0, 1])
def test_sort(name, desc):
    got = K.stable_order(_col(A[f"sort/in/{name}"]), bool(desc)).cpu().numpy()
    np.testing.assert_array_equal(got, A[f"sort/out/{name}/{desc}"])


def test_soft_path_with_tape_gradients():
    logits = A["soft/logits"]
    with Tape() as tape:
        x = tq.Tensor(logits)
        pe = tq.pe_encode(x)
        backward(reduce_sum(mul(pe.values, tq.tensor(A["soft/softmax_grad_in"]))))
        np.testing.assert_allclose(pe.values.numpy(), A["soft/softmax"], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(tape.gradient(x).numpy(), A["soft/softmax_grad"], rtol=1e-9,
                                   atol=1e-15)
    np.testing.assert_array_equal(tq.pe_decode(pe).values.numpy(), A["soft/pe_decode"])
    p1, p2, w, Gm = A["soft/p1"], A["soft/p2"], A["soft/w"], A["soft/G"]
    n = p1.shape[0]
    for agg in ("count", "sum", "avg"):
        with Tape() as tape:
            a, b, v = tq.Tensor(p1), tq.Tensor(p2), tq.Tensor(w)
            res = tq.soft_groupby([tq.EncodedTensor(a, tq.ProbabilityEncoding(3)),
                                   tq.EncodedTensor(b, tq.ProbabilityEncoding(4))], agg,
                                  v if agg != "count" else None)
            backward(reduce_sum(mul(res.counts, tq.tensor(Gm))))
            np.testing.assert_allclose(res.counts.numpy(), A[f"soft/{agg}/grid"], rtol=1e-9,
                                       atol=n * 2.0**-31)
            np.testing.assert_allclose(tape.gradient(a).numpy(), A[f"soft/{agg}/dp1"], rtol=1e-8,
                                       atol=1e-9)
            np.testing.assert_allclose(tape.gradient(b).numpy(), A[f"soft/{agg}/dp2"], rtol=1e-8,
                                       atol=1e-9)
            if agg != "count":
                np.testing.assert_allclose(tape.gradient(v).numpy(), A[f"soft/{agg}/dw"], rtol=1e-8,
                                           atol=1e-9)
    with Tape() as tape:
        pb = tq.Tensor(p2)
        res = tq.soft_groupby([tq.one_hot_pe(A["soft/onehot_codes"], 6),
                               tq.EncodedTensor(pb, tq.ProbabilityEncoding(4))])
        backward(reduce_sum(mul(res.counts, tq.tensor(A["soft/onehot/G"]))))
        np.testing.assert_allclose(res.counts.numpy(), A["soft/onehot/grid"], atol=n * 2.0**-31)
        np.testing.assert_allclose(tape.gradient(pb).numpy(), A["soft/onehot/dp"], rtol=1e-12)
    sc = tq.soft_count(tq.EncodedTensor(tq.tensor([[0.9, 0.1], [0.2, 0.8], [0.7, 0.3]]),
                                        tq.ProbabilityEncoding(2)))
    np.testing.assert_allclose(sc.numpy(), A["spec/soft_count"], atol=3 * 2.0**-31)


def test_tpch_end_to_end_through_sql():
    from paper_2211_02753_b200 import workloads as wl

    li = {k.split("/")[-1]: A[k] for k in A.files if k.startswith("tpch/in/")}
    cat = tq.Catalog()
    cat.register("lineitem", wl.lineitem_table(li))
    for q, sql, reg in (("q1", wl.Q1_SQL, wl.q1_registry()), ("q6", wl.Q6_SQL, wl.q6_registry())):
        plan = tq.lower(tq.bind(tq.parse(sql), cat, reg))
        cq = tq.compile_plan(plan, tq.CompileConfig(), reg)
        assert tq.explain(plan) == META["plans"][q]["explain"]
        assert cq.explain_compiled() == META["plans"][q]["compiled"]
        res = cq.run(cat)
        assert list(res.schema.names) == META["plans"][q]["names"]
        for name, col in zip(res.schema.names, res.columns):
            got, exp = col.values.numpy(), A[f"tpch/{q}/{name}"]
            assert got.dtype == exp.dtype
            if exp.dtype.kind == "f":
                np.testing.assert_allclose(got, exp, rtol=1e-9)
            else:
                np.testing.assert_array_equal(got, exp)


def test_gather_vjp_golden():
    """take_rows / gather VJP (tq/tensor.py:609-612): tdp_scatter_add_rows,
    duplicate indices accumulate like np.add.at."""
    from paper_2211_02753_b200.tensor import gather

    src, idx, w = A["gather/src"], A["gather/idx"], A["gather/w"]
    with Tape() as tape:
        a = tq.Tensor(src)
        out = gather(a, tq.Tensor(idx.astype(np.int64)), axis=0)
        backward(reduce_sum(mul(out, tq.tensor(w))))
        np.testing.assert_array_equal(out.numpy(), A["gather/out"])
        np.testing.assert_allclose(tape.gradient(a).numpy(), A["gather/grad"], rtol=1e-12,
                                   atol=1e-14)


def _score_query(X, W0, sql, n_rows):
    from paper_2211_02753_b200.storage import FLOAT
    from paper_2211_02753_b200.tensor import reshape

    lin = tq.Linear(X.shape[1], 1, np.random.default_rng(8), name="sc", dtype="float64")
    if W0 is not None:
        np.testing.assert_array_equal(lin.weight.value.numpy(), W0)  # same Glorot init
    reg = tq.UdfRegistry()
    reg.register(tq.UdfEntry("sc", (("s", FLOAT),), 1,
                             lambda c: (tq.plain(reshape(lin(c.values), (n_rows,))),),
                             lin.parameters, pe_outputs=False))
    cat = tq.Catalog()
    cat.register_tensor(tq.Tensor(X), "T")
    q = tq.compile_plan(tq.lower(tq.bind(tq.parse(sql), cat, reg)),
                        tq.CompileConfig(trainable=True), reg)
    return q, cat, lin


def _run_score(q, cat, lin, G):
    from paper_2211_02753_b200.tensor import add

    res = q.run(cat)
    loss = tq.tensor(0.0)
    for j, col in enumerate(res.columns[:2]):
        loss = add(loss, reduce_sum(mul(col.values, tq.tensor(G[j:j + 1]))))
    backward(loss)
    out = [c.values.numpy() for c in res.columns]
    dW = q.tape.gradient(lin.weight.value).numpy()
    db = q.tape.gradient(lin.bias.value).numpy()
    q.end_session()
    return out, dW, db


def test_global_soft_aggregates_golden():
    """GlobalAggSoftOp (tq/compiler.py:265-288) forward and tape gradients,
    with and without a WHERE (filter -> take_rows -> gather VJP), against the
    reference's own run."""
    X = A["globsoft/X"]
    for tag in ("filtered", "plain"):
        sql = META["globsoft"][tag]["sql"]
        q, cat, lin = _score_query(X, A["globsoft/W"], sql, X.shape[0])
        assert q.explain_compiled() == META["globsoft"][tag]["compiled"]
        out, dW, db = _run_score(q, cat, lin, A[f"globsoft/{tag}/G"])
        for got, nm in zip(out, META["globsoft"][tag]["names"]):
            exp = A[f"globsoft/{tag}/{nm}"]
            assert got.dtype == exp.dtype, nm
            np.testing.assert_allclose(got, exp, rtol=1e-9, err_msg=nm)
        np.testing.assert_allclose(dW, A[f"globsoft/{tag}/dW"], rtol=1e-9)
        np.testing.assert_allclose(db, A[f"globsoft/{tag}/db"], rtol=1e-9)


def test_global_soft_aggregates_large_vs_oracle():
    """The same chain at 300k rows (native column sums, scatter-add VJP over
    ~150k gathered rows) against the oracle's closed form."""
    from oracle import relational as orc

    rng = np.random.default_rng(4)
    X = rng.normal(size=(300_001, 6))
    G = np.array([0.7, -1.3])
    for sql, thr in (("SELECT SUM(s), AVG(s), COUNT(*) FROM (SELECT s FROM sc(T) WHERE s > 0.05)",
                      0.05), ("SELECT SUM(s), AVG(s), COUNT(*) FROM sc(T)", None)):
        q, cat, lin = _score_query(X, None, sql, X.shape[0])
        out, dW, db = _run_score(q, cat, lin, G)
        W, b = lin.weight.value.numpy(), lin.bias.value.numpy()
        s, avg, cnt, edW, edb = orc.score_global_soft(X, W, b, thr, G)
        np.testing.assert_allclose(out[0], s, rtol=1e-9)
        np.testing.assert_allclose(out[1], avg, rtol=1e-9)
        np.testing.assert_array_equal(out[2], cnt)
        np.testing.assert_allclose(dW, edW, rtol=1e-9)
        np.testing.assert_allclose(db, edb, rtol=1e-9)

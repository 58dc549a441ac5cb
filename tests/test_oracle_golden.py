"""CPU: pin the oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  Integer / index results bit-exact, float
results to the last few ulps (same numpy operations)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import relational as orc
from oracle import tpch as otpch

G = Path(__file__).resolve().parent / "golden"
A = np.load(G / "golden.npz")
META = json.loads((G / "golden.json").read_text())


def test_filter_cases():
    names = ["i64", "f64", "f32", "big"]
    cols = [A[f"filter/col/{k}"] for k in names]
    for ci, preds in enumerate(META["filter_cases"]):
        p = [(names.index(c), op, lit) for c, op, lit in preds]
        out = orc.filter_exact(cols, p)
        for k, o in zip(names, out):
            np.testing.assert_array_equal(o, A[f"filter/{ci}/{k}"], err_msg=f"case {ci} {preds}")


def test_dictionary_filter_cases():
    codes = A["dictfilter/codes"]
    entries = META["dictfilter"]["entries"]
    for ci, (op, lit) in enumerate(META["dictfilter"]["cases"]):
        idx = orc.filter_indices([codes], [(0, op, lit)], {0: entries})
        np.testing.assert_array_equal(codes[idx], A[f"dictfilter/{ci}"])


def test_groupby_and_global():
    k1, k2 = A["groupby/in/k1"], A["groupby/in/k2"]
    vf, vf32, vi = A["groupby/in/vf"], A["groupby/in/vf32"], A["groupby/in/vi"]
    aggs = [("count", None), ("sum", vf), ("avg", vf), ("sum", vf32), ("avg", vf32),
            ("sum", vi), ("avg", vi)]
    keys, out = orc.groupby_exact([k1, k2], aggs)
    for j, kv in enumerate(keys):
        np.testing.assert_array_equal(kv, A[f"groupby/out/key{j}"])
    for j, o in enumerate(out):
        exp = A[f"groupby/out/agg{j}"]
        assert o.dtype == exp.dtype
        np.testing.assert_array_equal(o, exp)
    g = orc.global_aggregate(len(vf), aggs)
    for j, o in enumerate(g):
        exp = A[f"global/out/{j}"]
        assert o.dtype == exp.dtype
        np.testing.assert_array_equal(o, exp)
    e = orc.global_aggregate(0, [("count", None), ("sum", vf[:0]), ("avg", vf[:0])])
    for j, o in enumerate(e):
        np.testing.assert_array_equal(o, A[f"global/empty/{j}"])
        assert o.dtype == A[f"global/empty/{j}"].dtype


def test_spec_examples():
    keys, aggs = orc.groupby_exact([np.array([1, 1, 2]), np.array([0, 1, 0])], [("count", None)])
    np.testing.assert_array_equal(np.stack(keys), A["spec/groupby/keys"])
    np.testing.assert_array_equal(aggs[0], A["spec/groupby/counts"])
    np.testing.assert_array_equal(A["spec/groupby/keys"], [[1, 1, 2], [0, 1, 0]])
    out = orc.sort_limit([np.array([0.2, 0.9, 0.5]), np.arange(3)], 0, True, 2)
    np.testing.assert_array_equal(out[1], A["spec/sort_limit"])
    np.testing.assert_array_equal(A["spec/sort_limit"], [1, 2])
    np.testing.assert_array_equal(orc.stable_order(np.array([1, 0, 1, 0]), True), A["spec/desc_ties"])
    np.testing.assert_array_equal(A["spec/desc_ties"], [0, 2, 1, 3])
    np.testing.assert_allclose(orc.soft_groupby([np.array([[0.9, 0.1], [0.2, 0.8], [0.7, 0.3]])]),
                               A["spec/soft_count"])
    np.testing.assert_allclose(A["spec/soft_count"], [1.8, 1.2])
    np.testing.assert_array_equal(orc.dense_exact_counts([np.array([0, 1, 1, 2]),
                                                          np.array([1, 0, 1, 1])], [3, 2]),
                                  A["spec/dense_exact_counts"])


@pytest.mark.parametrize("name", ["i64", "f64"])
@pytest.mark.parametrize("desc", [0, 1])
def test_sort(name, desc):
    np.testing.assert_array_equal(orc.stable_order(A[f"sort/in/{name}"], bool(desc)),
                                  A[f"sort/out/{name}/{desc}"])


def test_soft_path():
    logits = A["soft/logits"]
    p = orc.softmax(logits)
    np.testing.assert_allclose(p, A["soft/softmax"], rtol=1e-14, atol=1e-16)
    np.testing.assert_allclose(orc.softmax_vjp(p, A["soft/softmax_grad_in"]), A["soft/softmax_grad"],
                               rtol=1e-12, atol=1e-15)
    np.testing.assert_array_equal(orc.pe_decode(p), A["soft/pe_decode"])
    p1, p2, w, G_ = A["soft/p1"], A["soft/p2"], A["soft/w"], A["soft/G"]
    for agg in ("count", "sum", "avg"):
        grid = orc.soft_groupby([p1, p2], agg, w if agg != "count" else None)
        np.testing.assert_allclose(grid, A[f"soft/{agg}/grid"], rtol=1e-12, atol=1e-14)
    (d1, d2), _ = orc.soft_groupby_vjp([p1, p2], G_)
    np.testing.assert_allclose(d1, A["soft/count/dp1"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(d2, A["soft/count/dp2"], rtol=1e-12, atol=1e-14)
    (d1, d2), dw = orc.soft_groupby_vjp([p1, p2], G_, w)
    np.testing.assert_allclose(d1, A["soft/sum/dp1"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(dw, A["soft/sum/dw"], rtol=1e-12, atol=1e-14)
    codes = A["soft/onehot_codes"]
    oh = orc.one_hot(codes, 6)
    np.testing.assert_allclose(orc.soft_groupby([oh, p2]), A["soft/onehot/grid"], rtol=1e-12)
    (_, dp), _ = orc.soft_groupby_vjp([oh, p2], A["soft/onehot/G"])
    np.testing.assert_allclose(dp, A["soft/onehot/dp"], rtol=1e-12, atol=1e-14)


def test_tpch_end_to_end():
    li = {k.split("/")[-1]: A[k] for k in A.files if k.startswith("tpch/in/")}
    q1 = otpch.q1(li)
    for name in META["plans"]["q1"]["names"]:
        np.testing.assert_allclose(q1[name], A[f"tpch/q1/{name}"], rtol=1e-12)
        assert q1[name].dtype == A[f"tpch/q1/{name}"].dtype
    q6 = otpch.q6(li)
    np.testing.assert_allclose(q6["sum_rev"], A["tpch/q6/sum_rev"], rtol=1e-12)


def test_llp_closed_form_matches_reference_tape():
    X, bag, target = A["llp/X"], A["llp/bag"], A["llp/target"]
    W, b = A["llp/W4"], A["llp/b4"]
    loss, grid, dW, db = orc.llp_forward_backward(X, bag, W, b, target, 25)
    np.testing.assert_allclose(grid, A["llp/grid5"], rtol=1e-12)
    np.testing.assert_allclose(dW, A["llp/dW5"], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(db, A["llp/db5"], rtol=1e-10, atol=1e-14)


def test_join_oracle_vs_nested_loop():
    rng = np.random.default_rng(5)
    for _ in range(20):
        probe = rng.integers(0, 10, size=rng.integers(0, 40))
        build = rng.integers(0, 10, size=rng.integers(0, 40))
        a = orc.join_inner(probe, build)
        b = orc.join_nested_loop(probe, build)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])


def test_gather_vjp_and_global_soft_golden():
    src, idx, w = A["gather/src"], A["gather/idx"], A["gather/w"]
    np.testing.assert_array_equal(src[idx], A["gather/out"])
    np.testing.assert_allclose(orc.gather_rows_vjp(src.shape, idx, w), A["gather/grad"],
                               rtol=1e-13, atol=1e-14)
    X, W, b = A["globsoft/X"], A["globsoft/W"], A["globsoft/b"]
    for tag, thr in (("filtered", 0.05), ("plain", None)):
        s, avg, cnt, dW, db = orc.score_global_soft(X, W, b, thr, A[f"globsoft/{tag}/G"])
        np.testing.assert_allclose(s, A[f"globsoft/{tag}/sum_s"], rtol=1e-12)
        np.testing.assert_allclose(avg, A[f"globsoft/{tag}/avg_s"], rtol=1e-12)
        np.testing.assert_array_equal(cnt, A[f"globsoft/{tag}/count"])
        np.testing.assert_allclose(dW, A[f"globsoft/{tag}/dW"], rtol=1e-12)
        np.testing.assert_allclose(db, A[f"globsoft/{tag}/db"], rtol=1e-12)

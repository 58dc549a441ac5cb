"""CPU: host-side logic of the drop-in boundary (no kernel launches).

API surface, SQL front end and plan dumps vs the reference's golden output,
compile-time rules, error classes, and the C-ABI library's exported symbols.
"""

from __future__ import annotations

import json
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200 import _native
from paper_2211_02753_b200 import workloads as wl

ROOT = Path(__file__).resolve().parent.parent
META = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())

REFERENCE_ALL = [
    "AdamState", "BindError", "Catalog", "ColumnType", "CompileConfig", "CompileError",
    "CompiledQuery", "DictionaryEncoding", "EncodedTensor", "EncodingError", "GroupedCounts",
    "KernelError", "Linear", "MLP", "Parameter", "PlainEncoding", "PrivacyParams",
    "ProbabilityEncoding", "Schema", "SqlSyntaxError", "StorageError", "StringDictionary", "Table",
    "Tape", "Tensor", "TensorError", "TrainConfig", "TrainError", "UdfEntry", "UdfRegistry",
    "adam_step", "backward", "bind", "classifier_tvf", "compile_plan", "compile_query", "create",
    "dict_decode", "dict_encode", "explain", "export", "grad_check", "laplace_noise", "lower",
    "make_scoring_udf", "mse_loss", "one_hot_pe", "parse", "pe_decode", "pe_encode", "plain",
    "sgd_step", "soft_count", "soft_groupby", "table_from_columns", "tensor", "to_sql", "train",
]


def test_public_api_matches_reference():
    assert sorted(tq.__all__) == sorted(REFERENCE_ALL)
    for name in REFERENCE_ALL:
        assert hasattr(tq, name), name


def _lineitem_catalog(rows=100):
    cat = tq.Catalog()
    cat.register("lineitem", wl.lineitem_table(wl.lineitem_arrays(0.001, rows=rows)))
    return cat


@pytest.mark.parametrize("q,sql,reg", [("q1", wl.Q1_SQL, wl.q1_registry),
                                       ("q6", wl.Q6_SQL, wl.q6_registry)])
def test_plans_match_reference_golden(q, sql, reg):
    cat = _lineitem_catalog()
    r = reg()
    ast = tq.parse(sql)
    assert tq.to_sql(ast) == META["plans"][q]["to_sql"]
    assert tq.parse(tq.to_sql(ast)) == ast
    plan = tq.lower(tq.bind(ast, cat, r))
    assert tq.explain(plan) == META["plans"][q]["explain"]
    cq = tq.compile_plan(plan, tq.CompileConfig(), r)
    assert cq.explain_compiled() == META["plans"][q]["compiled"]
    assert list(cq.output_names) == META["plans"][q]["names"]


def test_syntax_errors_carry_offsets():
    with pytest.raises(tq.SqlSyntaxError, match=r"at offset 7 \(expected identifier\)"):
        tq.parse("SELECT FROM t")
    with pytest.raises(tq.SqlSyntaxError, match="unterminated string"):
        tq.parse('SELECT * FROM t WHERE a = "x')
    with pytest.raises(tq.SqlSyntaxError, match="LIMIT needs an integer"):
        tq.parse("SELECT * FROM t LIMIT 1.5")
    with pytest.raises(tq.SqlSyntaxError, match="trailing input"):
        tq.parse("SELECT * FROM t t2")


def test_bind_errors():
    cat = _lineitem_catalog()
    reg = tq.UdfRegistry()
    with pytest.raises(tq.BindError, match="did you mean 'l_tax'"):
        tq.bind(tq.parse("SELECT l_taxx FROM lineitem"), cat, reg)
    with pytest.raises(tq.BindError, match="is string but literal"):
        tq.bind(tq.parse("SELECT * FROM lineitem WHERE l_returnflag = 3"), cat, reg)
    with pytest.raises(tq.BindError, match="not an aggregate and not in GROUP BY"):
        tq.bind(tq.parse("SELECT l_tax, COUNT(*) FROM lineitem GROUP BY l_returnflag"), cat, reg)
    with pytest.raises(tq.BindError, match="SUM needs a numeric column"):
        tq.bind(tq.parse("SELECT SUM(l_returnflag) FROM lineitem"), cat, reg)


def test_trainable_rejects_sort_and_plain_keys():
    cat = _lineitem_catalog()
    reg = tq.UdfRegistry()
    plan = tq.lower(tq.bind(tq.parse("SELECT * FROM lineitem ORDER BY l_tax"), cat, reg))
    with pytest.raises(tq.CompileError, match="Sort has no differentiable"):
        tq.compile_plan(plan, tq.CompileConfig(trainable=True), reg)
    plan = tq.lower(tq.bind(tq.parse("SELECT l_returnflag, COUNT(*) FROM lineitem GROUP BY l_returnflag"),
                            cat, reg))
    with pytest.raises(tq.CompileError, match="probability-encoded keys"):
        tq.compile_plan(plan, tq.CompileConfig(trainable=True), reg)


def test_cpu_device_is_rejected():
    cat = _lineitem_catalog()
    reg = tq.UdfRegistry()
    plan = tq.lower(tq.bind(tq.parse("SELECT COUNT(*) FROM lineitem"), cat, reg))
    q = tq.compile_plan(plan, tq.CompileConfig(device="cpu"), reg)
    with pytest.raises(tq.CompileError, match="not executable"):
        q.run(cat)


def test_udf_registry_rules():
    reg = tq.UdfRegistry()
    e = tq.UdfEntry("f", (("x", tq.ColumnType("float")),), 1, lambda c: (c,), ())
    reg.register(e)
    with pytest.raises(tq.KernelError, match="already registered"):
        reg.register(e)
    with pytest.raises(tq.KernelError, match="unknown function"):
        reg.invoke("g", [])


def test_kernels_refuse_host_tensors():
    """No CPU fallback: a relational kernel on host tensors fails loudly."""
    from paper_2211_02753_b200.kernels import groupby_exact, stable_order

    col = tq.plain(tq.Tensor(np.arange(10)))
    if col.values.data.is_cuda:
        pytest.skip("GPU present")
    with pytest.raises(_native.NativeError, match="CUDA"):
        stable_order(col)
    with pytest.raises(_native.NativeError, match="CUDA"):
        groupby_exact([col], [("count", None)])


def _header_symbols() -> list[str]:
    text = (ROOT / "include" / "tdp_kernels.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tdp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _native.load()
    syms = _header_symbols()
    assert len(syms) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.library_path())],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tdp_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert sorted(_native.exported_symbols()) == syms
    for s in syms:
        getattr(lib, s)
    assert lib.tdp_version().startswith(b"tdp-b200")


def test_pipeline_codegen_compiles_q1_program_with_nvrtc():
    """The fused Q1 kernel's source is generated and compiled for sm_100a
    (NVRTC needs no GPU); checks the generated code's structure."""
    import ctypes

    import torch

    from paper_2211_02753_b200.lazy import Expr, Pred, Program, Selection

    a = wl.lineitem_arrays(0.0001, rows=64)
    t = {k: torch.from_numpy(v) for k, v in a.items()}
    prog = Program()
    rf, ls = Expr.column(t["l_returnflag"]), Expr.column(t["l_linestatus"])
    p, d, tx, q = (Expr.column(t[c]) for c in ("l_extendedprice", "l_discount", "l_tax", "l_quantity"))
    one = Expr.const(1.0, "float64")
    dp = Expr("mul", "float64", (p, Expr("sub", "float64", (one, d))))
    ch = Expr("mul", "float64", (dp, Expr("add", "float64", (one, tx))))
    sel = Selection(64, [Pred(t["l_shipdate"], "<=", _native.CMP_I64, 10471, 0.0)], torch.device("cpu"))
    keys = [_native.Key(prog.value(rf), 0, 0, 3), _native.Key(prog.value(ls), 0, 0, 2)]
    aggs = [_native.Agg(_native.AGG_SUM_F64, prog.value(e)) for e in (q, p, dp, ch, d)]
    aggs.append(_native.Agg(_native.AGG_COUNT, 0))
    preds, npreds = prog.predicates(sel)
    buf = ctypes.create_string_buffer(1 << 16)
    rc = _native.load().tdp_pipeline_codegen(
        _native.columns(prog.cols, False), len(prog.cols), 64, preds, npreds, prog.native_instrs(),
        len(prog.instrs), _native.struct_array(_native.Key, keys), 2,
        _native.struct_array(_native.Agg, aggs), len(aggs), None, 0, 1, buf, len(buf))
    assert rc > 0, _native.last_error()
    src = buf.value.decode()
    assert "#define TDP_G 6" in src and "#define TDP_NF 5" in src
    assert "#define TDP_ACCMODE 1" in src  # 36 cells -> shared-memory accumulator columns
    assert "tdp_bulk_load(sb + 0u" in src  # column tiles stream through the bulk-copy ring
    # the UDF's (1 - d) and (1 + t) become SSA values; (1.0) is shared (CSE)
    assert src.count("P.imf[") == 2  # once in tdp_eval, once in tdp_project


def test_pipeline_codegen_packs_exact_decimal_sums_of_compact_q1():
    """On compact storage (int32 cents, int8 hundredths, measured value ranges)
    Q1's five float sums are restated as exact scaled-integer programs
    (c*(100-d), c*(100-d)*(100+t)) and, with the row count, packed into three
    64-bit shared-memory words per thread and group (pipeline.cu
    convert_decimal_sums / pack_fields)."""
    import ctypes

    import torch

    from paper_2211_02753_b200.compact import decode_expr
    from paper_2211_02753_b200.lazy import Expr, Pred, Program, Selection, set_value_range

    n = 60_000_000  # SF10: 2048 rows per thread at most -> 12-bit count field

    def col(dt, lo, hi, div):
        x = torch.empty(n, dtype=dt)
        set_value_range(x, lo, hi)
        return decode_expr(x, div)

    rf, ls = (decode_expr(torch.empty(n, dtype=torch.uint8), 0) for _ in range(2))
    q, p = col(torch.int8, 1, 50, 1), col(torch.int32, 90000, 10494950, 100)
    d, tx = col(torch.int8, 0, 10, 100), col(torch.int8, 0, 8, 100)
    one = Expr.const(1.0, "float64")
    dp = Expr("mul", "float64", (p, Expr("sub", "float64", (one, d))))
    ch = Expr("mul", "float64", (dp, Expr("add", "float64", (one, tx))))
    prog = Program()
    sel = Selection(n, [Pred(torch.empty(n, dtype=torch.int16), "<=", _native.CMP_I64, 10471, 0.0)],
                    torch.device("cpu"))
    keys = [_native.Key(prog.value(rf), 0, 0, 3), _native.Key(prog.value(ls), 0, 0, 2)]
    aggs = [_native.Agg(_native.AGG_SUM_F64, prog.value(e)) for e in (q, p, dp, ch, d)]
    aggs.append(_native.Agg(_native.AGG_COUNT, 0))
    preds, npreds = prog.predicates(sel)
    buf = ctypes.create_string_buffer(1 << 17)
    rc = _native.load().tdp_pipeline_codegen(
        _native.columns(prog.cols, False), len(prog.cols), n, preds, npreds, prog.native_instrs(),
        len(prog.instrs), _native.struct_array(_native.Key, keys), 2,
        _native.struct_array(_native.Agg, aggs), len(aggs), None, 0, 1, buf, len(buf))
    assert rc > 0, _native.last_error()
    src = buf.value.decode()
    assert "#define TDP_NF 0" in src and "#define TDP_NI 5" in src  # all five sums exact
    assert "#define TDP_NW 3" in src and "#define TDP_SM_ROWS 21" in src  # 3 x (6 + reject slot)
    eval_body = src[src.index("bool tdp_eval"):src.index("tdp_smem_add")]
    assert "tdp_decimal" not in eval_body.split("slot = sl;")[1]  # q[] are integers
    add = src[src.index("void tdp_smem_add"):src.index("void tdp_smem_flush")]
    assert add.count(" * TDP_ACC_THREADS] += ") == 3  # three packed words per row
    # without measured ranges (int32/int8 type ranges) a CTA's sum of
    # c*(100-d)*(100+t) could exceed int64: that sum stays a float64 cell
    for t in prog.cols:
        if hasattr(t, "_tdp_range"):
            del t._tdp_range
    prog2 = Program()
    keys = [_native.Key(prog2.value(rf), 0, 0, 3), _native.Key(prog2.value(ls), 0, 0, 2)]
    aggs = [_native.Agg(_native.AGG_SUM_F64, prog2.value(e)) for e in (q, p, dp, ch, d)]
    aggs.append(_native.Agg(_native.AGG_COUNT, 0))
    preds, npreds = prog2.predicates(sel)
    rc = _native.load().tdp_pipeline_codegen(
        _native.columns(prog2.cols, False), len(prog2.cols), n, preds, npreds,
        prog2.native_instrs(), len(prog2.instrs), _native.struct_array(_native.Key, keys), 2,
        _native.struct_array(_native.Agg, aggs), len(aggs), None, 0, 0, buf, len(buf))
    assert rc > 0, _native.last_error()
    src2 = buf.value.decode()
    assert re.findall(r"#define TDP_(?:NF|NI|NW) \d+", src2) == [
        "#define TDP_NF 1", "#define TDP_NI 4", "#define TDP_NW 3"]


def test_trainable_order_by_is_rejected_without_soft_sort():
    """tq/compiler.py:464-475: Sort / Limit in trainable mode raise CompileError
    unless the soft-sort extension is asked for (CompileConfig.soft_sort_tau)."""
    import paper_2211_02753_b200 as tq
    from paper_2211_02753_b200.compiler import CompileError

    cat = tq.Catalog()
    reg = tq.UdfRegistry()
    cat.register_tensor(tq.Tensor(np.zeros((4, 3))), "T")
    reg.register(tq.make_scoring_udf("scorer", tq.Tensor(np.ones(3)), 1.0))
    plan = tq.lower(tq.bind(tq.parse("SELECT Score FROM scorer(T) ORDER BY Score LIMIT 2"), cat,
                            reg))
    with pytest.raises(CompileError, match="Sort has no differentiable implementation"):
        tq.compile_plan(plan, tq.CompileConfig(trainable=True), reg)
    q = tq.compile_plan(plan, tq.CompileConfig(trainable=True, soft_sort_tau=0.5), reg)
    assert "sort[soft]" in q.explain_compiled()

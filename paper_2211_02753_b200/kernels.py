"""Relational operator kernels (exact and soft) and the UDF/TVF registry.

Drop-in for ``tensorquery.kernels`` (tq/kernels.py): same functions, argument
meaning, output contracts and error classes/messages.  Every row-proportional
loop runs in libtdp_kernels.so (sm_100a) -- there is no CPU implementation:

==========================  =====================================================
reference (tq/kernels.py)   B200 path
==========================  =====================================================
comparison_mask  :54        tdp_filter_mask
filter_exact     :87        lazy Selection (tdp_filter_select when materialised)
take_rows        :44        tdp_gather_rows / tdp_scatter_add_rows (VJP)
groupby_exact    :108       fused tdp_scan_aggregate (dense keys) or
                            tdp_unique_inverse + tdp_groupby_codes (general)
_global_aggregate (compiler.py:206)  fused tdp_scan_aggregate, no keys
soft_count       :183       tdp_soft_groupby_fwd/bwd (one dense key)
soft_groupby     :212       tdp_soft_groupby_fwd/bwd (dense + compact one-hot keys)
dense_exact_counts :238     tdp_groupby_codes
stable_order     :256       tdp_sort_order (LSD radix, numpy stable semantics)
sort_limit / limit_rows     tdp_sort_order + tdp_gather_rows
equi_join (new)             tdp_join_prepare / tdp_join_emit
==========================  =====================================================
"""

from __future__ import annotations

import os
from ctypes import c_int32, c_void_p
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np
import torch

from . import _native as nat
from . import hostread
from .hostread import read_int, read_ints
from .autograd import (SoftKeySpec, gather_many, gather_rows_raw, linear_keys,
                       soft_groupby_grid, soft_linear_count, soft_linear_supported,
                       chunked_soft_linear_count)
from .encodings import (
    DecodedArgmax,
    DecodedCodes,
    EncodedTensor,
    EncodingError,
    OneHotValue,
    onehot_payload,
    plain,
    trusted,
)
from .lazy import (
    native_predicates,
    DeferredCount,
    Expr,
    PrefixRows,
    LazyValue,
    Pred,
    Program,
    Selection,
    as_expr,
    base_rows,
    compact_source,
    decimal_predicates,
    resolve_predicate,
)
from .distributed import (
    allgather_rows,
    allreduce_sum,
    allreduce_partials,
    allreduce_ranges,
    current_group,
    exchange_rows,
    is_sharded,
    key_destination,
    world_size,
)
from .storage import ColumnType
from .tensor import (
    FLOAT_DTYPES,
    Parameter,
    Tensor,
    _finish,
    _grad_mode,
    _inputs,
    active_tape,
    add,
    div,
    dtype_name,
    gather,
    slice_axis,
    pending_softmax,
    mul,
    reshape,
    tensor,
    to_device,
    torch_dtype,
)

AVG_STABILIZER = 1e-12
DENSE_SLOT_LIMIT = 1 << 16


class KernelError(ValueError):
    """Kernel precondition violation (types, shapes, arity)."""


def _as_index(indices) -> torch.Tensor:
    if isinstance(indices, Tensor):
        indices = indices.data
    return to_device(indices if isinstance(indices, torch.Tensor) else np.asarray(indices, dtype=np.int64)).to(torch.int64).reshape(-1)


# ---------------------------------------------------------------------------
# Row selection shared by filter / sort / limit
# ---------------------------------------------------------------------------


def take_rows(col: EncodedTensor, indices) -> EncodedTensor:
    """Compact a column to the given row indices, preserving gradients."""
    idx = _as_index(indices)
    v = col.values
    oh = onehot_payload(v)
    with trusted():
        if oh is not None:
            return EncodedTensor(Tensor(OneHotValue(gather_rows_raw(oh.codes, idx), oh.k, oh.dtype)),
                                 col.encoding)
        if v.dtype in FLOAT_DTYPES and active_tape() is not None:
            return EncodedTensor(gather(v, Tensor(idx), axis=0), col.encoding)
        return EncodedTensor(Tensor(gather_rows_raw(v.data, idx)), col.encoding)


def take_rows_many(columns: Sequence[EncodedTensor], indices) -> list[EncodedTensor]:
    """take_rows of several columns by one index vector: the plain ones in a
    single gather launch (tdp_gather_rows over up to 16 columns)."""
    idx = _as_index(indices)
    out: list = [None] * len(columns)
    plain = []
    for i, c in enumerate(columns):
        v = c.values
        if onehot_payload(v) is None and not (v.dtype in FLOAT_DTYPES and active_tape() is not None):
            plain.append(i)
        else:
            out[i] = take_rows(c, idx)
    for b in range(0, len(plain), 16):
        part = plain[b:b + 16]
        got = gather_many([columns[i].values.data for i in part], idx)
        with trusted():
            for i, g in zip(part, got):
                out[i] = EncodedTensor(Tensor(g), columns[i].encoding)
    return out


_OPS = ("=", "<>", "<", ">", "<=", ">=")


def _resolve(col: EncodedTensor, op: str, literal, base: Optional[torch.Tensor],
             divisor: int = 0) -> Pred:
    """Validate one comparison exactly as comparison_mask does and resolve it.

    ``divisor`` > 0: ``base`` holds the column as scaled integers (a compact
    float64 column, compact.py); the float64 comparison becomes a decimal one
    on the stored integers (decode by the same division, then compare)."""
    if op not in _OPS:
        raise KernelError(f"unknown comparison operator {op!r}")
    if col.is_dictionary():
        if not isinstance(literal, str):
            raise KernelError(f"string column compared against {literal!r}")
        code = col.encoding.dictionary.code_of(literal)
        if code is None:
            return Pred(None, op, nat.CMP_NONE, 0, 0.0)
        return Pred(base, op, nat.CMP_I64, code, 0.0)
    if col.is_pe():
        raise KernelError("cannot filter on a probability-encoded column")
    if isinstance(literal, str):
        raise KernelError(f"numeric column compared against string {literal!r}")
    if col.values.ndim != 1:
        raise KernelError("filters require scalar columns")
    cmp, li, lf = resolve_predicate(col.values.dtype, op, literal)
    if divisor and cmp == nat.CMP_F64:
        raise KernelError("decimal column predicates resolve through _resolve_all")
    return Pred(base if cmp in (nat.CMP_I64, nat.CMP_F64, nat.CMP_F32) else None, op, cmp, li, lf)


def _resolve_all(col: EncodedTensor, op: str, literal, base: Optional[torch.Tensor],
                 divisor: int = 0) -> list[Pred]:
    """_resolve, with predicates on compact decimal columns rewritten into
    int64 comparisons on the stored integers (lazy.decimal_predicates)."""
    if divisor and not col.is_dictionary() and not col.is_pe() and op in _OPS \
            and not isinstance(literal, str) and col.values.ndim == 1:
        cmp, _, lf = resolve_predicate(col.values.dtype, op, literal)
        if cmp == nat.CMP_F64:
            out = []
            for o, c, li in decimal_predicates(op, lf, divisor):
                keep = c in (nat.CMP_I64, nat.CMP_DEC)
                out.append(Pred(base if keep else None, o, c, li, lf))
            return out
    return [_resolve(col, op, literal, base)]


def comparison_mask(col: EncodedTensor, op: str, literal) -> torch.Tensor:
    """Boolean row mask for ``col <op> literal`` (tdp_filter_mask)."""
    data = col.values.data if not col.is_pe() else None
    p = _resolve(col, op, literal, data)
    n = col.row_count
    out = torch.empty(n, dtype=torch.bool, device=data.device if data is not None else None)
    cols = [data] if p.col is not None else []
    if n:
        nat.require_cuda(out, *cols)
        nat.call("tdp_filter_mask", nat.columns(cols), len(cols),
                 native_predicates([p], {id(c): i for i, c in enumerate(cols)}), 1, n,
                 nat.ptr(out), nat.stream())
    return out


def _row_space(columns: Sequence[EncodedTensor]) -> Optional[tuple[Optional[Selection], int]]:
    """Common (selection, base rows) of columns that can stay lazy, else None."""
    sel_id, sel, n = None, None, None
    for c in columns:
        v = c.values
        if v._t is not None:
            s, rows = None, (int(v._t.shape[0]) if v._t.dim() else -1)
        elif isinstance(v._lazy, LazyValue):
            s = v._lazy.sel
            rows = s.n if s is not None else base_rows(v._lazy.expr)
        else:
            return None
        key = id(s) if s is not None else None
        if n is None:
            sel_id, sel, n = key, s, rows
        elif key != sel_id or rows != n:
            return None
    return sel, (n if n is not None else 0)


def filter_exact(columns: Sequence[EncodedTensor],
                 predicates: Sequence[tuple[int, str, object]]) -> list[EncodedTensor]:
    """Conjunctive filter: AND of per-predicate masks, then row compaction.

    The compaction is late: the returned columns are lazy views of the input
    rows under the new selection; consumers either fuse it (group-by) or
    materialise it with tdp_filter_select + tdp_gather_rows.
    """
    if not columns:
        return []
    space = _row_space(columns) if active_tape() is None else None
    if space is None:
        return _filter_eager(columns, predicates)
    sel, n = space
    preds = []
    for idx, op, literal in predicates:
        col = columns[idx]
        v = col.values
        base, divisor = None, 0
        if not col.is_pe() and v.ndim == 1:
            if v._t is not None:
                base = v._t
            elif v._lazy.expr.op == "col":
                base = v._lazy.expr.col
            elif compact_source(v._lazy.expr) is not None:  # compact storage
                base, divisor = compact_source(v._lazy.expr)
            else:  # predicate on a computed column: evaluate eagerly
                return _filter_eager(columns, predicates)
        preds.extend(_resolve_all(col, op, literal, base, divisor))
    device = _device_of([as_expr(c.values)[0] for c in columns], sel)
    new_sel = sel.refine(preds) if sel is not None else Selection(n, preds, device)
    out = []
    for c in columns:
        v = c.values
        if v._t is not None:
            lv = LazyValue(Expr.column(v._t), new_sel, valid_for=c.encoding)
        else:
            lv = LazyValue(v._lazy.expr, new_sel, valid_for=c.encoding)
        with trusted():
            out.append(EncodedTensor(Tensor(lv), c.encoding))
    return out


def _filter_eager(columns: Sequence[EncodedTensor], predicates) -> list[EncodedTensor]:
    n = columns[0].row_count
    preds = []
    cols: list[torch.Tensor] = []
    index: dict[int, int] = {}
    for idx, op, literal in predicates:
        col = columns[idx]
        data = None
        if not col.is_pe() and (col.is_dictionary() or not isinstance(literal, str)):
            data = col.values.data.detach() if col.values.ndim == 1 else None
        p = _resolve(col, op, literal, data)
        if p.col is not None and id(p.col) not in index:
            index[id(p.col)] = len(cols)
            cols.append(p.col)
        preds.append(p)
    sel = Selection(n, preds, cols[0].device if cols else None)
    if not cols:
        sel._run()
    idx = sel.indices()
    return [take_rows(c, idx) for c in columns]


# ---------------------------------------------------------------------------
# Exact group-by (tq/kernels.py:108-167) and global aggregates (compiler.py:206)
# ---------------------------------------------------------------------------

AggInput = tuple[str, Optional[object]]  # ("count", None) | ("sum"/"avg", values)


def _value_dtype(v) -> str:
    if isinstance(v, Tensor):
        return v.dtype
    if isinstance(v, torch.Tensor):
        return dtype_name(v)
    return np.asarray(v).dtype.name


def _as_value(v):
    if isinstance(v, (Tensor, torch.Tensor)):
        return v
    return Tensor(np.asarray(v))


def _agg_kind(func: str, dtype: str) -> int:
    if func == "count":
        return nat.AGG_COUNT
    return nat.AGG_SUM_F64 if dtype in FLOAT_DTYPES else nat.AGG_SUM_I64


def _emit_kinds(agg_specs, kinds) -> "c_int32 * n":
    """Kinds for a group-by emit call: AVG aggregates carry TDP_AGG_AVG_BIT,
    so the emit kernel writes the float64 mean (no cast / divide launches)."""
    ek = [k | nat.AGG_AVG_BIT if f == "avg" else k for (f, _), k in zip(agg_specs, kinds)]
    return (c_int32 * max(1, len(ek)))(*ek)


def _fusable(values: Sequence) -> Optional[tuple[Optional[Selection], int]]:
    """Common selection / base length of all operands, or None."""
    sel_key, sel, n = 0, None, None
    for v in values:
        e, s = as_expr(v)
        rows = s.n if s is not None else base_rows(e)
        if rows < 0:
            return None
        k = id(s) if s is not None else None
        if n is None:
            sel_key, sel, n = k, s, rows
        elif k != sel_key or rows != n:
            return None
    return sel, (n or 0)


def _materialize(v) -> torch.Tensor:
    if isinstance(v, Tensor):
        return v.data.detach()
    return to_device(v)


def _scan_aggregate(exprs_keys: Sequence[Expr], spans: Sequence[tuple[int, int]],
                    aggs: Sequence[tuple[int, Optional[Expr]]], sel: Optional[Selection],
                    n: int, device, avg_mask: Optional[int] = None):
    """Run tdp_scan_aggregate; returns (counts[G], sums_raw[naggs, G] int64 bits, G).

    With ``avg_mask`` (an unsharded group-by) the finalisation runs in the
    same native call (tdp_scan_aggregate_grouped) and the result is
    ``(out_keys[nkeys, G], out_counts[G], out_aggs[naggs, G], out_groups[1])``
    in tdp_groupby_finalize's layout."""
    prog = Program()
    keys = [nat.Key(prog.value(e), 0, lo, span) for e, (lo, span) in zip(exprs_keys, spans)]
    agg_structs = []
    for kind, e in aggs:
        if kind == nat.AGG_COUNT:
            agg_structs.append(nat.Agg(kind, 0))
        else:
            val = prog.value(e if kind == nat.AGG_SUM_F64 or e.dtype == "int64" else e.cast("int64"))
            agg_structs.append(nat.Agg(kind, val))
    preds, npreds = prog.predicates(sel)
    slots = 1
    for _, span in spans:
        slots *= span
    nat.require_cuda(*prog.cols)
    # one allocation: counts [slots] | sums [naggs, slots] | workspace
    na = max(1, len(aggs))
    ws_words = (int(nat.load().tdp_scan_aggregate_workspace(n, slots, len(aggs))) + 7) // 8
    buf = torch.empty(slots * (1 + na) + ws_words, dtype=torch.int64, device=device)
    counts = buf[:slots]
    sums = buf[slots:slots * (1 + na)].view(na, slots)
    ws = buf[slots * (1 + na):]
    hook = PROFILE_HOOK
    if hook is not None:
        hook.begin("tdp_scan_aggregate", n)
    if avg_mask is not None:
        nk = max(1, len(keys))
        fin = torch.empty((nk + 1 + na) * slots + 1, dtype=torch.int64, device=device)
        out_keys = fin[:nk * slots].view(nk, slots)
        out_counts = fin[nk * slots:(nk + 1) * slots]
        out_aggs = fin[(nk + 1) * slots:(nk + 1 + na) * slots].view(na, slots)
        out_groups = fin[(nk + 1 + na) * slots:]
        nat.call("tdp_scan_aggregate_grouped", prog.native_columns(), len(prog.cols), n, preds,
                 npreds, prog.native_instrs(), len(prog.instrs), nat.struct_array(nat.Key, keys),
                 len(keys), nat.struct_array(nat.Agg, agg_structs), len(agg_structs),
                 nat.ptr(counts), nat.ptr(sums), nat.ptr(ws), ws.numel() * 8, avg_mask,
                 nat.ptr(out_keys), nat.ptr(out_counts), nat.ptr(out_aggs), nat.ptr(out_groups),
                 nat.stream())
        if hook is not None:
            hook.end("tdp_scan_aggregate")
        return out_keys, out_counts, out_aggs, out_groups
    nat.call("tdp_scan_aggregate", prog.native_columns(), len(prog.cols), n, preds, npreds,
             prog.native_instrs(), len(prog.instrs), nat.struct_array(nat.Key, keys), len(keys),
             nat.struct_array(nat.Agg, agg_structs), len(agg_structs), nat.ptr(counts),
             nat.ptr(sums), nat.ptr(ws), ws.numel() * 8, nat.stream())
    if hook is not None:
        hook.end("tdp_scan_aggregate")
    return counts, sums, slots


# Optional kernel timer (bench.py): object with begin(name, rows) / end(name)
# that records CUDA events on the current stream around native calls.
PROFILE_HOOK = None


def _finalize(counts, sums, slots, spans, aggs_kinds, avg_mask, device, defer_rows=False):
    nkeys = len(spans)
    keys = nat.struct_array(nat.Key, [nat.Key(0, 0, lo, span) for lo, span in spans])
    aggs = nat.struct_array(nat.Agg, [nat.Agg(k, 0) for k in aggs_kinds])
    nk, na = max(1, nkeys), max(1, len(aggs_kinds))
    buf = torch.empty((nk + 1 + na) * slots + 1, dtype=torch.int64, device=device)
    out_keys = buf[:nk * slots].view(nk, slots)
    out_counts = buf[nk * slots:(nk + 1) * slots]
    out_aggs = buf[(nk + 1) * slots:(nk + 1 + na) * slots].view(na, slots)
    out_groups = buf[(nk + 1 + na) * slots:]
    nat.call("tdp_groupby_finalize", nat.ptr(counts), nat.ptr(sums), slots, keys, nkeys, aggs,
             len(aggs_kinds), avg_mask, nat.ptr(out_keys), nat.ptr(out_counts), nat.ptr(out_aggs),
             nat.ptr(out_groups), nat.stream())
    if defer_rows:  # padded [slots] outputs + the occupied count, read by the host later
        return out_keys, out_counts, out_aggs, DeferredCount(out_groups)
    g = read_int(out_groups)
    return out_keys[:, :g], out_counts[:g], out_aggs[:, :g], g


def _agg_outputs(aggs: Sequence[tuple[str, str]], raw: torch.Tensor, counts: torch.Tensor,
                 already_avg: bool) -> list[torch.Tensor]:
    """Typed aggregate columns from raw 8-byte results (views, no copies:
    result columns are immutable)."""
    out = []
    for a, (func, dt) in enumerate(aggs):
        r = raw[a]
        if func == "count":
            out.append(r)
        elif func == "avg":
            if already_avg:
                out.append(r.view(torch.float64))
            else:
                s = r.view(torch.float64) if dt in FLOAT_DTYPES else r.to(torch.float64)
                out.append(s / counts.to(torch.float64))
        else:
            out.append(r.view(torch.float64) if dt in FLOAT_DTYPES else r)
    return out


def groupby_exact(keys: Sequence[EncodedTensor], aggs: Sequence[AggInput], *,
                  defer_rows: bool = False) -> tuple[list, list]:
    """Group rows by the key columns and aggregate.

    Returns key-value arrays and aggregate arrays over the non-empty groups,
    ordered by ascending combined key (lexicographic over the key columns).
    With ``defer_rows`` (the compiler's GroupAggExactOp) the dense fused path
    returns :class:`~.lazy.PrefixRows` payloads instead of torch tensors: the
    number of occupied groups stays on the device until the host reads it, so
    the query does not synchronise.
    """
    if not keys:
        raise KernelError("groupby_exact requires at least one key column")
    for k in keys:
        if k.is_pe():
            raise KernelError("exact group-by cannot consume PE keys; decode first")
        if k.values.ndim != 1 or k.values.dtype != "int64":
            raise KernelError(
                f"group-by keys must be integer or dictionary columns, got {k.values.dtype}"
            )
    key_vals = [k.values for k in keys]
    agg_specs: list[tuple[str, str]] = []
    agg_vals: list = []
    for func, values in aggs:
        if func == "count":
            agg_specs.append(("count", "int64"))
            agg_vals.append(None)
            continue
        if values is None:
            raise KernelError(f"{func} aggregate needs a value column of {keys[0].row_count} rows")
        if func not in ("sum", "avg"):
            raise KernelError(f"unknown aggregate {func!r}")
        v = _as_value(values)
        agg_specs.append((func, _value_dtype(v)))
        agg_vals.append(v)

    fused = _groupby_decoded_linear(keys, agg_specs, defer_rows)
    if fused is not None:
        return fused
    operands = key_vals + [v for v in agg_vals if v is not None]
    space = _fusable(operands)
    if space is not None and all(as_expr(k)[0].op in ("col", "cast", "add", "sub", "mul", "neg", "square")
                                 for k in key_vals):
        return _groupby_fused(keys, key_vals, agg_specs, agg_vals, space, defer_rows)
    return _groupby_general(keys, key_vals, agg_specs, agg_vals)


def _groupby_decoded_linear(keys, agg_specs, defer_rows=False):
    """COUNT grouped by pe_decode(pe_encode(Linear(X))) and decoded one-hot
    codes -- the exact swap of a trained LLP query -- in
    one pass over X (tdp_linear_argmax_count), then the dense finalisation of
    the fused group-by (occupied groups in ascending key order).  None when
    the keys / aggregates do not have that form."""
    if not agg_specs or any(f != "count" for f, _ in agg_specs):
        return None
    if active_tape() is not None or current_group() is not None:
        return None
    dense, kinds, codes = None, [], []
    for j, k in enumerate(keys):
        v = k.values
        lz = v._lazy if v._t is None else None
        if isinstance(lz, DecodedArgmax) and lz._out is None and dense is None:
            dense = (j, lz)
            kinds.append(("dense", lz.k))
        elif isinstance(lz, DecodedCodes):
            kinds.append(("onehot", lz.k))
            codes.append(lz.codes.contiguous())
        else:
            return None
    if dense is None:
        return None
    pos, dec = dense
    lin = dec.pend.lin
    spec = SoftKeySpec(kinds)
    if not soft_linear_supported(lin.x, lin.w, spec.cells):
        return None
    nat.require_cuda(*codes)
    x, w = lin.x.detach().contiguous(), lin.w.detach().contiguous()
    b = None if lin.b is None else lin.b.detach().contiguous()
    n, d = x.shape
    slots = spec.cells
    counts = torch.empty(slots, dtype=torch.int64, device=x.device)
    nat.call("tdp_linear_argmax_count", nat.ptr(x), nat.TORCH_TO_TDP[x.dtype], n, d,
             int(w.shape[1]), nat.ptr(w), nat.ptr(b), linear_keys(spec, pos, codes),
             len(kinds), pos, nat.ptr(counts), nat.stream())
    naggs = len(agg_specs)
    sums = counts.unsqueeze(0).expand(naggs, slots).contiguous()
    spans = [(0, kk) for _, kk in kinds]
    kinds_native = [nat.AGG_COUNT] * naggs
    out_keys, out_counts, out_aggs, g = _finalize(counts, sums, slots, spans, kinds_native, 0,
                                                  x.device, defer_rows)
    key_values = [out_keys[j].contiguous() for j in range(len(keys))]
    agg_values = _agg_outputs(agg_specs, out_aggs, out_counts, already_avg=True)
    if defer_rows:
        return ([PrefixRows(kv, g) for kv in key_values], [PrefixRows(a, g) for a in agg_values])
    return key_values, agg_values


def _groupby_fused(keys, key_vals, agg_specs, agg_vals, space, defer_rows=False):
    sel, n = space
    kexprs = [as_expr(v)[0] for v in key_vals]
    device = _device_of(kexprs, sel)
    spans: list[tuple[int, int]] = []
    need_range = [j for j, k in enumerate(keys) if not k.is_dictionary()]
    ranges: dict[int, tuple[int, int]] = {}
    runs = False
    if need_range:
        if any(kexprs[j].op != "col" for j in need_range):
            return _groupby_general(keys, key_vals, agg_specs, agg_vals)
        prog = Program()
        kc = [prog.col_index(kexprs[j].col) for j in need_range]
        preds, npreds = prog.predicates(sel)
        group = current_group()
        # one int64 key, no predicates, not sharded: also check whether the
        # key column is sorted in short runs (the sorted-runs group-by)
        check_runs = (len(keys) == 1 and npreds == 0 and group is None
                      and prog.cols[kc[0]].dtype == torch.int64)
        mm = torch.empty(2 * len(need_range) + (2 if check_runs else 0), dtype=torch.int64,
                         device=device)
        nat.require_cuda(*prog.cols)
        nat.call("tdp_scan_minmax_runs", prog.native_columns(), len(prog.cols), n, preds, npreds,
                 (c_int32 * len(kc))(*kc), len(kc), nat.ptr(mm),
                 nat.ptr(mm[2:]) if check_runs else None, nat.stream())
        if group is not None:
            lo, hi = allreduce_ranges(mm[0::2].contiguous(), mm[1::2].contiguous(), group)
            mm = torch.stack([lo, hi], dim=1).reshape(-1)
        host = read_ints(mm)
        runs = check_runs and host[2] == 0 and host[3] == 0
        for t, j in enumerate(need_range):
            ranges[j] = (host[2 * t], host[2 * t + 1])
        if any(lo > hi for lo, hi in ranges.values()):
            return _empty_groups(len(keys), agg_specs, device)
    slots = 1
    for j, k in enumerate(keys):
        if k.is_dictionary():
            lo, span = 0, max(1, len(k.encoding.dictionary))
        else:
            lo, hi = ranges[j]
            span = hi - lo + 1
        spans.append((lo, span))
        slots *= span
    if slots > DENSE_SLOT_LIMIT:  # high cardinality: sort-based (sharded: all-to-all)
        return _groupby_general(keys, key_vals, agg_specs, agg_vals,
                                key_range=ranges.get(0) if len(keys) == 1 else None,
                                runs=runs)
    agg_exprs = []
    for (func, dt), v in zip(agg_specs, agg_vals):
        kind = _agg_kind(func, dt)
        agg_exprs.append((kind, as_expr(v)[0] if v is not None else None))
    avg_mask = 0
    for a, (func, _) in enumerate(agg_specs):
        if func == "avg":
            avg_mask |= 1 << a
    group = current_group()
    if not is_sharded(group):  # scan + reduce + finalise in one call
        out_keys, out_counts, out_aggs, out_groups = _scan_aggregate(
            kexprs, spans, agg_exprs, sel, n, device, avg_mask=avg_mask)
        if defer_rows:
            g = DeferredCount(out_groups)
        else:
            g = read_int(out_groups)
            out_keys, out_counts, out_aggs = out_keys[:, :g], out_counts[:g], out_aggs[:, :g]
    else:
        counts, sums, slots = _scan_aggregate(kexprs, spans, agg_exprs, sel, n, device)
        allreduce_partials(counts, sums, [a for a, (k, _) in enumerate(agg_exprs)
                                          if k == nat.AGG_SUM_F64], group,
                           tuple(a for a, (k, _) in enumerate(agg_exprs) if k == nat.AGG_COUNT))
        kinds = [k for k, _ in agg_exprs]
        out_keys, out_counts, out_aggs, g = _finalize(counts, sums, slots, spans, kinds, avg_mask,
                                                      device, defer_rows)
    key_values = [out_keys[j].contiguous() for j in range(len(keys))]
    agg_values = _agg_outputs(agg_specs, out_aggs, out_counts, already_avg=True)
    if defer_rows:
        return ([PrefixRows(k, g) for k in key_values], [PrefixRows(a, g) for a in agg_values])
    return key_values, agg_values


def _device_of(exprs, sel):
    if sel is not None and sel.device is not None:
        return sel.device
    stack = list(exprs)
    while stack:
        e = stack.pop()
        if e.op == "col":
            return e.col.device
        stack.extend(e.args)
    return torch.device("cuda")


def _empty_groups(nkeys: int, agg_specs, device):
    key_values = [torch.empty(0, dtype=torch.int64, device=device) for _ in range(nkeys)]
    outs = []
    for func, dt in agg_specs:
        if func == "count":
            outs.append(torch.empty(0, dtype=torch.int64, device=device))
        elif func == "avg" or dt in FLOAT_DTYPES:
            outs.append(torch.empty(0, dtype=torch.float64, device=device))
        else:
            outs.append(torch.empty(0, dtype=torch.int64, device=device))
    return key_values, outs


def unique_inverse(key: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """np.unique(key, return_inverse=True) on the device (tdp_unique_inverse)."""
    key = key.contiguous().to(torch.int64)
    nat.require_cuda(key)
    n = key.numel()
    dev = key.device
    uniques = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    inverse = torch.empty(n, dtype=torch.int64, device=dev)
    count = torch.empty(1, dtype=torch.int64, device=dev)
    lib = nat.load()
    ws = nat.workspace(lib.tdp_sort_workspace(n) + 2 * ((n * 8 + 255) // 256 * 256) + 1024, dev)
    nat.call("tdp_unique_inverse", nat.ptr(key), n, nat.ptr(uniques), nat.ptr(inverse),
             nat.ptr(count), nat.ptr(ws), ws.numel(), nat.stream())
    u = read_int(count) if n else 0
    return uniques[:u], inverse


def _groupby_codes(codes: torch.Tensor, slots: int, agg_specs, agg_vals, n: int, device):
    kinds = [_agg_kind(f, dt) for f, dt in agg_specs]
    vals = []
    keep = []
    for (func, dt), v, kind in zip(agg_specs, agg_vals, kinds):
        if kind == nat.AGG_COUNT:
            vals.append(None)
            continue
        t = _materialize(v)
        if t.dim() != 1 or t.shape[0] != n:
            raise KernelError(f"{func} aggregate needs a value column of {n} rows")
        if t.dtype == torch.bool:
            t = t.to(torch.int64)
        keep.append(t)
        vals.append(t)
    cols = (nat.Column * max(1, len(vals)))()
    for a, t in enumerate(vals):
        cols[a] = nat.column(t) if t is not None else nat.Column(None, nat.I64, 0, 0, 1)
    counts = torch.empty(slots, dtype=torch.int64, device=device)
    sums = torch.empty((max(1, len(kinds)), slots), dtype=torch.int64, device=device)
    nat.require_cuda(codes)
    ws = nat.workspace(nat.load().tdp_groupby_codes_workspace(
        slots, sum(k == nat.AGG_SUM_F64 for k in kinds)), device)
    nat.call("tdp_groupby_codes", nat.ptr(codes), n, slots, cols,
             (c_int32 * max(1, len(kinds)))(*kinds), len(kinds), nat.ptr(counts), nat.ptr(sums),
             nat.ptr(ws), ws.numel(), nat.stream())
    return counts, sums


def _groupby_general(keys, key_vals, agg_specs, agg_vals, key_range=None, runs=False):
    """Sort-based path (the reference's np.unique algorithm on the device);
    hash / bitmap aggregation for one high-cardinality int64 key."""
    kdata = [_materialize(v) for v in key_vals]
    n = int(kdata[0].shape[0])
    vdata = []
    for (func, dt), v in zip(agg_specs, agg_vals):
        if v is None:
            vdata.append(None)
            continue
        t = _materialize(v)
        if t.dim() != 1 or t.shape[0] != n:
            raise KernelError(f"{func} aggregate needs a value column of {n} rows")
        vdata.append(t)
    nat.require_cuda(*kdata)
    group = current_group()
    if is_sharded(group):
        return _groupby_sharded(kdata, agg_specs, vdata, group)
    return _groupby_local(kdata, agg_specs, vdata, key_range, runs)


def _lex_order(keys: Sequence[torch.Tensor]) -> torch.Tensor:
    """Stable lexicographic order of key tuples (LSD over the key columns)."""
    order = None
    for k in reversed(list(keys)):
        kk = k if order is None else gather_rows_raw(k, order)
        o = stable_order(plain(Tensor(kk)))
        order = o if order is None else gather_rows_raw(order, o)
    return order


def _groupby_sharded(kdata, agg_specs, vdata, group):
    """High-cardinality group-by across ranks: repartition rows by key with
    an NCCL all-to-all, group locally (every group now lives on one rank),
    all-gather the (small) results and order them by key."""
    world = world_size(group)
    device = kdata[0].device
    dest = key_destination(kdata, world)
    order = stable_order(plain(Tensor(dest)))
    send_counts, _ = _groupby_codes(dest, world, [], [], int(dest.numel()), device)
    cols = [t.to(torch.int64) if t.dtype == torch.bool else t for t in list(kdata) +
            [v for v in vdata if v is not None]]
    recv = exchange_rows(gather_many(cols, order), send_counts, group)
    rk = recv[:len(kdata)]
    rv = iter(recv[len(kdata):])
    rvals = [None if v is None else next(rv) for v in vdata]
    key_values, aggs = _groupby_local(rk, agg_specs, rvals)
    allk = allgather_rows(list(key_values) + list(aggs), group)
    kv, av = allk[:len(key_values)], allk[len(key_values):]
    if kv[0].numel() == 0:
        return kv, av
    o = _lex_order(kv)
    return gather_many(kv, o), gather_many(av, o)


HASH_GROUPBY_MIN_ROWS = 1 << 16


# bitmap ranking of hash group-by keys while the key range is at most this many
# values per distinct key (beyond: radix sort of the distinct keys)
RANK_BITS_PER_GROUP = 1024


def _key_of_image(img: int) -> int:
    """int64 key of an order-preserving key image (key ^ INT64_MIN) read as int64."""
    u = (img & (2**64 - 1)) ^ (1 << 63)
    return u - (1 << 64) if u >= 1 << 63 else u


def _groupby_hash(key: torch.Tensor, agg_specs, agg_vals, n: int, device):
    """One int64 key, hash aggregation (tdp_groupby_hash_*): a pass over the
    rows instead of a sort of them; only the distinct keys are sorted."""
    kinds = [_agg_kind(f, dt) for f, dt in agg_specs]
    vals = []
    for (func, dt), v, kind in zip(agg_specs, agg_vals, kinds):
        if kind == nat.AGG_COUNT:
            vals.append(None)
            continue
        t = _materialize(v)
        if t.dim() != 1 or t.shape[0] != n:
            raise KernelError(f"{func} aggregate needs a value column of {n} rows")
        vals.append(t.to(torch.int64) if t.dtype == torch.bool else t.contiguous())
    cols = (nat.Column * max(1, len(vals)))()
    for a, t in enumerate(vals):
        cols[a] = nat.column(t) if t is not None else nat.Column(None, nat.I64, 0, 0, 1)
    kind_arr = (c_int32 * max(1, len(kinds)))(*kinds)
    key = key.contiguous()
    ws = nat.workspace(nat.load().tdp_groupby_hash_workspace(n, len(kinds)), device)
    info = torch.empty(3, dtype=torch.int64, device=device)
    nat.call("tdp_groupby_hash_prepare_ex", nat.ptr(key), n, cols, kind_arr, len(kinds),
             nat.ptr(info), nat.ptr(ws), ws.numel(), nat.stream())
    m, lo_img, hi_img = read_ints(info)  # group count and key range, one read
    keys_out = torch.empty(m, dtype=torch.int64, device=device)
    counts = torch.empty(m, dtype=torch.int64, device=device)
    sums = torch.empty((max(1, len(kinds)), m), dtype=torch.int64, device=device)
    key_range = ((hi_img - lo_img) & (2**64 - 1)) + 1 if m else 0
    if m and key_range <= min(RANK_BITS_PER_GROUP * m + (1 << 21), 1 << 32):
        # ascending key order by a bitmap rank over the range (a few
        # bandwidth-bound passes) instead of a radix sort of the m keys
        lo_key = _key_of_image(lo_img)
        rws = nat.workspace(nat.load().tdp_groupby_hash_rank_workspace(key_range), device)
        nat.call("tdp_groupby_hash_emit_ranked", n, _emit_kinds(agg_specs, kinds), len(kinds), m,
                 lo_key, key_range,
                 nat.ptr(keys_out), nat.ptr(counts), nat.ptr(sums), nat.ptr(ws), ws.numel(),
                 nat.ptr(rws), rws.numel(), nat.stream())
    else:
        nat.call("tdp_groupby_hash_emit", n, _emit_kinds(agg_specs, kinds), len(kinds), m,
                 nat.ptr(keys_out), nat.ptr(counts), nat.ptr(sums), nat.ptr(ws), ws.numel(),
                 nat.stream())
    return [keys_out], _agg_outputs(agg_specs, sums, counts, already_avg=True)


def _agg_columns(agg_specs, agg_vals, n: int):
    kinds = [_agg_kind(f, dt) for f, dt in agg_specs]
    vals = []
    for (func, dt), v, kind in zip(agg_specs, agg_vals, kinds):
        if kind == nat.AGG_COUNT:
            vals.append(None)
            continue
        t = _materialize(v)
        if t.dim() != 1 or t.shape[0] != n:
            raise KernelError(f"{func} aggregate needs a value column of {n} rows")
        vals.append(t.to(torch.int64) if t.dtype == torch.bool else t.contiguous())
    cols = (nat.Column * max(1, len(vals)))()
    for a, t in enumerate(vals):
        cols[a] = nat.column(t) if t is not None else nat.Column(None, nat.I64, 0, 0, 1)
    return kinds, vals, cols


def _groupby_bitmap(key: torch.Tensor, lo: int, span: int, agg_specs, agg_vals, n: int, device):
    """One int64 key in [lo, lo + span): bitmap-rank aggregation
    (tdp_groupby_bitmap_*) -- groups come out in ascending key order without
    a hash table or a sort; one host read (the group count)."""
    kinds, vals, cols = _agg_columns(agg_specs, agg_vals, n)
    kind_arr = (c_int32 * max(1, len(kinds)))(*kinds)
    key = key.contiguous()
    ws = nat.workspace(nat.load().tdp_groupby_bitmap_workspace(n, span, len(kinds)), device)
    info = torch.empty(1, dtype=torch.int64, device=device)
    nat.call("tdp_groupby_bitmap_prepare", nat.ptr(key), n, lo, span, cols, kind_arr, len(kinds),
             nat.ptr(info), nat.ptr(ws), ws.numel(), nat.stream())
    m = read_int(info)
    keys_out = torch.empty(m, dtype=torch.int64, device=device)
    counts = torch.empty(m, dtype=torch.int64, device=device)
    sums = torch.empty((max(1, len(kinds)), m), dtype=torch.int64, device=device)
    nat.call("tdp_groupby_bitmap_emit", n, lo, span, _emit_kinds(agg_specs, kinds), len(kinds), m,
             nat.ptr(keys_out), nat.ptr(counts), nat.ptr(sums), nat.ptr(ws), ws.numel(),
             nat.stream())
    return [keys_out], _agg_outputs(agg_specs, sums, counts, already_avg=True)


def _groupby_runs(key: torch.Tensor, agg_specs, agg_vals, n: int, device):
    """One int64 key column sorted in runs of <= 32 equal keys (checked by
    tdp_scan_minmax_runs): the runs are the groups (tdp_groupby_runs_*) --
    a count pass, a scan, an emit pass; sums in row order."""
    kinds, vals, cols = _agg_columns(agg_specs, agg_vals, n)
    key = key.contiguous()
    ws = nat.workspace(nat.load().tdp_groupby_runs_workspace(n), device)
    info = torch.empty(1, dtype=torch.int64, device=device)
    nat.call("tdp_groupby_runs_prepare", nat.ptr(key), n, nat.ptr(info), nat.ptr(ws), ws.numel(),
             nat.stream())
    m = read_int(info)
    keys_out = torch.empty(m, dtype=torch.int64, device=device)
    counts = torch.empty(m, dtype=torch.int64, device=device)
    sums = torch.empty((max(1, len(kinds)), m), dtype=torch.int64, device=device)
    nat.call("tdp_groupby_runs_emit", nat.ptr(key), n, cols, _emit_kinds(agg_specs, kinds),
             len(kinds), m, nat.ptr(keys_out), nat.ptr(counts), nat.ptr(sums), nat.ptr(ws),
             ws.numel(), nat.stream())
    return [keys_out], _agg_outputs(agg_specs, sums, counts, already_avg=True)


def _groupby_local(kdata, agg_specs, agg_vals, key_range=None, runs=False):
    device = kdata[0].device
    n = int(kdata[0].shape[0])
    if n == 0:
        return _empty_groups(len(kdata), agg_specs, device)
    if runs and len(kdata) == 1 and kdata[0].dtype == torch.int64:
        return _groupby_runs(kdata[0], agg_specs, agg_vals, n, device)
    if len(kdata) == 1 and kdata[0].dtype == torch.int64 and key_range is not None:
        span = key_range[1] - key_range[0] + 1
        if 1 <= span <= min(1 << 34, RANK_BITS_PER_GROUP * n + (1 << 21)):
            return _groupby_bitmap(kdata[0], key_range[0], span, agg_specs, agg_vals, n, device)
    if len(kdata) == 1 and kdata[0].dtype == torch.int64 and n >= HASH_GROUPBY_MIN_ROWS:
        return _groupby_hash(kdata[0], agg_specs, agg_vals, n, device)
    uniqs, codes = zip(*[unique_inverse(k) for k in kdata])
    if len(kdata) == 1:
        group_codes, slots = codes[0], int(uniqs[0].numel())
        key_values = [uniqs[0]]
    else:
        spaces = [max(1, int(u.numel())) for u in uniqs]
        combined = torch.zeros(n, dtype=torch.int64, device=device)
        for c, s in zip(codes, spaces):
            combined = combined * s + c
        occupied, group_codes = unique_inverse(combined)
        slots = int(occupied.numel())
        key_values = []
        rem = occupied.clone()
        for u, s in zip(reversed(uniqs), reversed(spaces)):
            key_values.append(gather_rows_raw(u, (rem % s).contiguous()))
            rem = rem // s
        key_values.reverse()
    counts, sums = _groupby_codes(group_codes, slots, agg_specs, agg_vals, n, device)
    return key_values, _agg_outputs(agg_specs, sums, counts, already_avg=False)


def global_aggregate(row_source: Sequence[EncodedTensor], agg_inputs) -> list[torch.Tensor]:
    """``_global_aggregate`` (tq/compiler.py:206-215): no GROUP BY.

    count -> int64 [rows]; sum -> [sum] in the input dtype; avg -> [mean]
    (float64 for int input, NaN when empty).  One fused pass computes the row
    count and every sum.
    """
    vals = [_as_value(v) for f, v in agg_inputs if f != "count"]
    operands = list(vals) + [c.values for c in row_source[:1]]
    space = _fusable(operands) if operands else None
    rows_dev = raw = None
    if space is not None:
        sel, n = space
        device = _device_of([as_expr(v)[0] for v in operands], sel)
        specs = [(nat.AGG_COUNT, None) if f == "count"
                 else (_agg_kind(f, _value_dtype(v)), as_expr(_as_value(v))[0])
                 for f, v in agg_inputs]
        rows_dev, raw, _ = _scan_aggregate([], [], specs, sel, n, device)
        allreduce_partials(rows_dev, raw, [a for a, (k, _) in enumerate(specs)
                                           if k == nat.AGG_SUM_F64], current_group(),
                           tuple(a for a, (k, _) in enumerate(specs) if k == nat.AGG_COUNT))
    elif current_group() is not None:
        raise KernelError("sharded global aggregate needs its inputs in one row space")
    out = []
    for a, (func, values) in enumerate(agg_inputs):
        if func == "count":
            if rows_dev is not None:
                out.append(rows_dev[:1].clone())
            else:
                out.append(torch.tensor([row_source[0].row_count if row_source else 0],
                                        dtype=torch.int64, device=_materialize(vals[0]).device
                                        if vals else None))
            continue
        v = _as_value(values)
        dt = _value_dtype(v)
        if raw is not None:
            r, cnt = raw[a, :1], rows_dev[:1]
        else:  # value columns in different row spaces: one pass per column
            cnt, r = _scan_single(_materialize(v))
        total = r.view(torch.float64) if dt in FLOAT_DTYPES else r
        if func == "sum":
            # numpy keeps the input dtype: float32 stays float32, bool -> any()
            out.append(total != 0 if dt == "bool" else total.to(torch_dtype(dt)).clone())
        else:
            mean = total.to(torch.float64) / cnt.to(torch.float64)
            # numpy: float32 mean stays float32; an empty input gives float64 NaN
            if dt == "float32" and read_int(cnt) > 0:
                mean = mean.to(torch.float32)
            out.append(mean)
    return out


def _scan_single(t: torch.Tensor):
    spec = [(nat.AGG_COUNT, None), (_agg_kind("sum", _value_dtype(t)), Expr.column(t.contiguous()))]
    counts, sums, _ = _scan_aggregate([], [], spec, None, int(t.shape[0]), t.device)
    return counts[:1], sums[1, :1]


# ---------------------------------------------------------------------------
# Soft aggregates over PE columns (tq/kernels.py:175-235)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class GroupedCounts:
    """Dense aggregate grid over the cross-product of the key spaces."""

    key_spaces: tuple[int, ...]
    counts: Tensor


def _soft_inputs(pes: Sequence[EncodedTensor]):
    kinds, tensors, dts = [], [], []
    tape = active_tape()
    for p in pes:
        oh = onehot_payload(p.values)
        if oh is not None:
            kinds.append(("onehot", oh.k))
            tensors.append(oh.codes)
            dts.append(oh.dtype)
        else:
            kinds.append(("dense", p.encoding.num_classes))
            t = tape.input_for(p.values) if tape is not None else p.values.data
            tensors.append(t.contiguous())
            dts.append(p.values.dtype)
    return SoftKeySpec(kinds), tensors, dts


def _soft_linear_count(pes: Sequence[EncodedTensor], spaces: tuple[int, ...]) -> Optional[Tensor]:
    """Soft count of one deferred ``pe_encode(Linear(X))`` key crossed with
    one-hot keys, in one fused pass over X (tdp_soft_linear_count_fwd; the
    backward recomputes P from X).  None when the keys do not have that form."""
    dense, kinds, dts, codes = None, [], [], []
    for j, p in enumerate(pes):
        oh = onehot_payload(p.values)
        if oh is not None:
            kinds.append(("onehot", oh.k))
            dts.append(oh.dtype)
            codes.append(oh.codes)
            continue
        pend = pending_softmax(p.values)
        if pend is None or dense is not None:
            return None
        dense = (j, pend, p.values.node)
        kinds.append(("dense", p.encoding.num_classes))
        dts.append(pend.dtype)
    if dense is None:
        return None
    pos, pend, node = dense
    if node is not None and node is not active_tape():
        return None
    lin = pend.lin
    spec = SoftKeySpec(kinds)
    chunked = getattr(lin, "wide", False)
    if not chunked and not soft_linear_supported(lin.x, lin.w, spec.cells):
        return None
    nat.require_cuda(*codes)
    joint_dt = dts[0]
    for d in dts[1:]:
        joint_dt = np.promote_types(joint_dt, d).name
    count = chunked_soft_linear_count if chunked else soft_linear_count
    with _grad_mode():
        grid = count(spec, pos, [c.contiguous() for c in codes], lin.x, lin.w, lin.b,
                     torch_dtype(joint_dt))
        grid = allreduce_sum(grid, current_group())  # row-sharded: global grid
        return _finish(grid.reshape(spaces))


def soft_count(pe: EncodedTensor) -> Tensor:
    """Differentiable count per class: column sums of the PE matrix."""
    if not pe.is_pe():
        raise EncodingError("soft_count requires a probability-encoded column")
    return soft_groupby([pe], "count").counts


def _joint_spaces(pes: Sequence[EncodedTensor]) -> tuple[tuple[int, ...], int]:
    if not pes:
        raise KernelError("soft_groupby requires at least one PE column")
    n = pes[0].row_count
    spaces = []
    for p in pes:
        if not p.is_pe():
            raise EncodingError("soft_groupby keys must be probability-encoded")
        if p.row_count != n:
            raise KernelError(f"soft_groupby keys disagree on row count ({p.row_count} vs {n})")
        spaces.append(p.encoding.num_classes)
    return tuple(spaces), n


def soft_groupby(pes: Sequence[EncodedTensor], agg: str = "count",
                 values: Optional[Tensor] = None) -> GroupedCounts:
    """Differentiable grouped aggregation over PE key columns.

    counts[c1..cm] = sum_i prod_j P_j[i, c_j]; every cell of the dense grid
    is emitted.  sum/avg weight each row's joint probability by a plain
    numeric column.  The n x prod(k) joint is never materialised.
    """
    spaces, n = _joint_spaces(pes)
    if agg == "count":
        fused = _soft_linear_count(pes, spaces)
        if fused is not None:
            return GroupedCounts(spaces, fused)
    spec, keys, dts = _soft_inputs(pes)
    nat.require_cuda(*keys)
    joint_dt = dts[0]
    for d in dts[1:]:
        joint_dt = np.promote_types(joint_dt, d).name
    with _grad_mode():
        grid = soft_groupby_grid(spec, keys, n, torch_dtype(joint_dt))
        grid = allreduce_sum(grid, current_group())  # row-sharded: global grid
        counts = _finish(grid.reshape(spaces))
    if agg == "count":
        return GroupedCounts(spaces, counts)
    if values is None:
        raise KernelError(f"soft {agg} needs a value column")
    if values.shape != (n,):
        raise KernelError(f"value column shape {list(values.shape)} != [{n}]")
    w = values if values.dtype in FLOAT_DTYPES else values.astype("float64")
    wdt = np.promote_types(joint_dt, w.dtype).name
    tape = active_tape()
    with _grad_mode():
        wt = tape.input_for(w) if tape is not None else w.data
        weighted_grid = soft_groupby_grid(spec, keys, n, torch_dtype(wdt), values=wt.contiguous())
        weighted_grid = allreduce_sum(weighted_grid, current_group())
        weighted = _finish(weighted_grid.reshape(spaces))
    if agg == "sum":
        return GroupedCounts(spaces, weighted)
    if agg == "avg":
        eps = tensor(AVG_STABILIZER, dtype=counts.dtype)
        return GroupedCounts(spaces, div(weighted, add(counts, eps)))
    raise KernelError(f"unknown soft aggregate {agg!r}")


def dense_exact_counts(codes: Sequence, spaces: Sequence[int]) -> torch.Tensor:
    """Exact contingency grid over fixed key spaces (densified group-by)."""
    spaces = tuple(int(s) for s in spaces)
    cs = [_as_index(c) for c in codes]
    n = int(cs[0].numel()) if cs else 0
    dev = cs[0].device if cs else None
    total = 1
    for s in spaces:
        total *= s
    if n:
        nat.require_cuda(*cs)
        from .encodings import _codes_out_of_range

        for c, s in zip(cs, spaces):
            if _codes_out_of_range(c, s):
                raise KernelError(f"key code out of range [0, {s})")
    combined = torch.zeros(n, dtype=torch.int64, device=dev)
    for c, s in zip(cs, spaces):
        combined = combined * s + c
    counts, _ = _groupby_codes(combined, max(1, total), [], [], n, dev)
    return counts[:total].reshape(spaces)


# ---------------------------------------------------------------------------
# Sort / limit (tq/kernels.py:256-280)
# ---------------------------------------------------------------------------


def stable_order(key: EncodedTensor, descending: bool = False) -> torch.Tensor:
    """Stable row order by a numeric or dictionary key (tdp_sort_order)."""
    if key.is_pe():
        raise KernelError("cannot sort by a probability-encoded column")
    if key.values.ndim != 1:
        raise KernelError("sort keys must be scalar columns")
    arr = key.values.data.detach()
    if arr.dtype == torch.bool:
        if descending:
            raise TypeError("The numpy boolean negative, the `-` operator, is not supported, "
                            "use the `~` operator or the logical_not function instead.")
        arr = arr.to(torch.int64)
    arr = arr.contiguous()
    nat.require_cuda(arr)
    n = int(arr.shape[0])
    out = torch.empty(n, dtype=torch.int64, device=arr.device)
    if n:
        ws = nat.workspace(nat.load().tdp_sort_workspace(n), arr.device)
        nat.call("tdp_sort_order", nat.columns([arr]), 1 if descending else 0, n, nat.ptr(out),
                 nat.ptr(ws), ws.numel(), nat.stream())
    return out


TOPK_MAX = 1024


def _sort_key_tensor(key: EncodedTensor, descending: bool) -> torch.Tensor:
    if key.is_pe():
        raise KernelError("cannot sort by a probability-encoded column")
    if key.values.ndim != 1:
        raise KernelError("sort keys must be scalar columns")
    arr = key.values.data.detach()
    if arr.dtype == torch.bool:
        if descending:
            raise TypeError("The numpy boolean negative, the `-` operator, is not supported, "
                            "use the `~` operator or the logical_not function instead.")
        arr = arr.to(torch.int64)
    arr = arr.contiguous()
    nat.require_cuda(arr)
    return arr


def topk_order(key: EncodedTensor, k: int, descending: bool = False) -> torch.Tensor:
    """``stable_order(key, descending)[:k]`` without ordering all rows
    (tdp_topk_order; 1 <= k <= TOPK_MAX)."""
    arr = _sort_key_tensor(key, descending)
    n = int(arr.shape[0])
    out = torch.empty(min(k, n), dtype=torch.int64, device=arr.device)
    if n:
        ws = nat.workspace(nat.load().tdp_topk_workspace(n, k), arr.device)
        nat.call("tdp_topk_order", nat.columns([arr]), 1 if descending else 0, n, k,
                 nat.ptr(out), nat.ptr(ws), ws.numel(), nat.stream())
    return out


def sort_limit(columns: Sequence[EncodedTensor], key_index: int,
               descending: bool = False, limit: Optional[int] = None) -> list[EncodedTensor]:
    """Stable order by one key, optionally truncated (tq/kernels.py:267-273);
    a small LIMIT takes the top rows without ordering the rest."""
    key = columns[key_index]
    if limit is not None and 0 < limit <= TOPK_MAX and limit < key.row_count:
        order = topk_order(key, limit, descending)
    else:
        order = stable_order(key, descending)
        if limit is not None:
            order = order[: max(0, limit)]
    return take_rows_many(columns, order)


def limit_rows(columns: Sequence[EncodedTensor], count: int) -> list[EncodedTensor]:
    if not columns:
        return []
    n = columns[0].row_count
    m = min(max(0, count), n)
    out = []
    with trusted():
        for c in columns:
            oh = onehot_payload(c.values)
            if oh is not None:
                out.append(EncodedTensor(Tensor(OneHotValue(oh.codes[:m], oh.k, oh.dtype)), c.encoding))
                continue
            v = c.values
            if v.dtype in FLOAT_DTYPES and active_tape() is not None:
                out.append(EncodedTensor(slice_axis(v, 0, 0, m), c.encoding))
            else:
                out.append(EncodedTensor(Tensor(v.data[:m]), c.encoding))
    return out


# ---------------------------------------------------------------------------
# Equi-join (builder-defined; the reference has none -- SURVEY §8 A20)
# ---------------------------------------------------------------------------


# dense-range join while the build key range is at most this many bits per
# build row (bitmap <= 8 B per build row, and <= 2^34 bits)
DENSE_JOIN_BITS_PER_ROW = 64


def column_range(t: torch.Tensor, compute: bool = True) -> Optional[tuple[int, int]]:
    """[min, max] of an int64 column: a column statistic cached on the tensor
    (valid while its in-place version is unchanged), like a zone map.
    Computed on first use with tdp_scan_minmax (one host read).  Inside a
    CUDA-graph capture the recorded run's answer is used (hostread.decision):
    the plan takes the same path; the dense join kernels still flag any key
    outside the range (a logged, device-checked read).  Gathered join outputs
    inherit their base column's range (a superset of theirs)."""
    return hostread.decision(lambda: _column_range(t, compute))


def _column_range(t: torch.Tensor, compute: bool) -> Optional[tuple[int, int]]:
    meta = getattr(t, "_tdp_range", None)
    if meta is not None and meta[0] == t._version:
        return meta[1], meta[2]
    if not compute or t.numel() == 0 or t.dtype != torch.int64 or t.dim() != 1 \
            or torch.cuda.is_current_stream_capturing():
        return None
    nat.require_cuda(t)
    prog = Program()
    kc = prog.col_index(t.contiguous())
    mm = torch.empty(2, dtype=torch.int64, device=t.device)
    preds, npreds = prog.predicates(None)
    nat.call("tdp_scan_minmax", prog.native_columns(), len(prog.cols), int(t.numel()), preds,
             npreds, (c_int32 * 1)(kc), 1, nat.ptr(mm), nat.stream())
    lo, hi = (int(v) for v in mm.tolist())
    t._tdp_range = (t._version, lo, hi)
    return lo, hi


def _inherit_range(out: torch.Tensor, base: torch.Tensor, compute: bool = False) -> None:
    if base.dtype != torch.int64 or base.dim() != 1:
        return
    r = column_range(base, compute=compute)
    if r is not None:
        out._tdp_range = (out._version, r[0], r[1])


def _dense_range(build_range, n_build: int) -> Optional[tuple[int, int]]:
    if build_range is None:
        return None
    lo, hi = build_range
    span = hi - lo + 1
    if span < 1 or span > min(1 << 34, DENSE_JOIN_BITS_PER_ROW * max(n_build, 1 << 16)):
        return None
    return lo, span


# Equi-join algorithm: "auto" = dense-range bitmap join when the build keys'
# range allows, else the hash join; "sort" = radix-sorted build +
# searchsorted probe (tdp_join_sorted_*, north_star's algorithm, measured
# slower on Q3 -- DESIGN.md §3.3).  Env TDP_JOIN_ALGO sets the default.
JOIN_ALGORITHM = os.environ.get("TDP_JOIN_ALGO", "auto")


def _join_sorted(pk: torch.Tensor, bk: torch.Tensor, probe_sel: Optional[Selection],
                 build_sel: Optional[Selection], predset):
    """Sort / searchsorted join; a filtered build side is compacted first
    (its selection's row ids), build rows are mapped back to base rows."""
    dev = pk.device
    bmap = None
    if build_sel is not None and build_sel.preds:
        bmap = build_sel.indices()
        bk = gather_rows_raw(bk, bmap)
    n_probe, n_build = int(pk.numel()), int(bk.numel())
    pc, npc, pp, npp = predset(probe_sel, n_probe, "probe")
    ws = nat.workspace(nat.load().tdp_join_sorted_workspace(n_build, n_probe), dev)
    cnt = torch.empty(1, dtype=torch.int64, device=dev)
    nat.call("tdp_join_sorted_prepare", nat.ptr(bk), n_build, nat.ptr(pk), n_probe, pc, npc, pp,
             npp, nat.ptr(cnt), nat.ptr(ws), ws.numel(), nat.stream())
    m = read_int(cnt)
    pi = torch.empty(m, dtype=torch.int64, device=dev)
    bi = torch.empty(m, dtype=torch.int64, device=dev)
    if m:
        nat.call("tdp_join_sorted_emit", nat.ptr(pk), n_build, n_probe, nat.ptr(pi), nat.ptr(bi),
                 nat.ptr(ws), ws.numel(), nat.stream())
    if bmap is not None:
        bi = gather_rows_raw(bmap, bi)
    return pi, bi


def join_indices(probe_key, build_key, probe_sel: Optional[Selection] = None,
                 build_sel: Optional[Selection] = None,
                 build_range: Optional[tuple[int, int]] = None, need_build_rows: bool = True
                 ) -> Optional[tuple[torch.Tensor, Optional[torch.Tensor]]]:
    """Inner equi-join row pairs: (probe rows, build rows), ordered by probe row
    then ascending build row (hash build, one probe per probe row).

    With ``probe_sel`` / ``build_sel`` a side is a filtered base relation: its
    key column is the *base* key column, the selection's predicates are
    evaluated inside the join's own passes, and the returned row ids of that
    side are base row ids (the filtered relation is never materialised).  One
    host synchronisation (the pair count) unless the build keys repeat; a
    filtered build with repeated keys returns None (the caller compacts the
    build side first).
    With ``build_range`` (every build key in [lo, hi], a column statistic)
    and a span small next to the build, the dense-range join runs first
    (bitmap instead of hash table; unique keys only -- repeated keys fall back
    to the hash join).  ``need_build_rows=False`` (no build column is output)
    returns None for the build rows when the build keys are unique."""
    pk = _materialize(probe_key).contiguous().to(torch.int64)
    bk = _materialize(build_key).contiguous().to(torch.int64)
    nat.require_cuda(pk, bk)
    dev = pk.device
    n_probe, n_build = int(pk.numel()), int(bk.numel())
    ws = nat.workspace(nat.load().tdp_join_workspace(n_build, n_probe), dev)
    info = torch.empty(2, dtype=torch.int64, device=dev)

    def predset(sel, n, what):
        if sel is None or not sel.preds:
            return nat.columns([]), 0, nat.struct_array(nat.Predicate, []), 0
        if sel.n != n:
            raise KernelError(f"{what} selection and key column disagree on row count")
        prog = Program()
        preds, npreds = prog.predicates(sel)
        nat.require_cuda(*prog.cols)
        return prog.native_columns(), len(prog.cols), preds, npreds

    if JOIN_ALGORITHM == "sort":
        return _join_sorted(pk, bk, probe_sel, build_sel, predset)
    bc, nbc, bp, nbp = predset(build_sel, n_build, "build")
    pc, npc, pp, npp = predset(probe_sel, n_probe, "probe")
    dense = _dense_range(build_range, n_build)
    if dense is not None and n_build and n_probe:
        lo, span = dense
        dws = nat.workspace(nat.load().tdp_join_dense_workspace(span, n_build, n_probe), dev)
        nat.call("tdp_join_dense_prepare", nat.ptr(bk), n_build, bc, nbc, bp, nbp, nat.ptr(pk),
                 n_probe, pc, npc, pp, npp, lo, span, int(need_build_rows), nat.ptr(info),
                 nat.ptr(dws), dws.numel(), nat.stream())
        m, fallback = read_ints(info)
        if not fallback:
            pi = torch.empty(m, dtype=torch.int64, device=dev)
            bi = torch.empty(m, dtype=torch.int64, device=dev) if need_build_rows else None
            if m:
                nat.call("tdp_join_dense_emit", nat.ptr(pk), n_build, n_probe, lo, span,
                         int(need_build_rows), nat.ptr(pi), nat.ptr(bi) if bi is not None else None,
                         nat.ptr(dws), dws.numel(), nat.stream())
            return pi, bi
    nat.call("tdp_join_prepare_ex", nat.ptr(bk), n_build, bc, nbc, bp, nbp, nat.ptr(pk), n_probe,
             pc, npc, pp, npp, 0, nat.ptr(info), nat.ptr(ws), ws.numel(), nat.stream())
    m, repeated = read_ints(info)
    if repeated:
        if nbp:
            return None
        nat.call("tdp_join_prepare_ex", nat.ptr(bk), n_build, bc, 0, bp, 0, nat.ptr(pk), n_probe,
                 pc, npc, pp, npp, 1, nat.ptr(info), nat.ptr(ws), ws.numel(), nat.stream())
        m = read_int(info[:1])
    pi = torch.empty(m, dtype=torch.int64, device=dev)
    bi = torch.empty(m, dtype=torch.int64, device=dev)
    if m:
        nat.call("tdp_join_emit", nat.ptr(pk), n_build, n_probe, nat.ptr(pi), nat.ptr(bi),
                 nat.ptr(ws), ws.numel(), nat.stream())
    return pi, bi


def _side_sources(cols: Sequence[EncodedTensor]):
    """(base tensors, selection or None) for one join side.

    Lazy views of one selection are read straight from their base columns
    (the probe side through the filtered probe pass, the build side through
    ``selection.indices()``); the filtered relation is never materialised.
    Anything else is materialised first (selection None)."""
    sels = set()
    for c in cols:
        v = c.values
        if v._t is not None or not isinstance(v._lazy, LazyValue) or v._lazy.expr.op != "col" \
                or v._lazy.sel is None:
            sels = None
            break
        sels.add(id(v._lazy.sel))
    if sels is not None and len(sels) == 1:
        sel = cols[0].values._lazy.sel
        return [c.values._lazy.expr.col for c in cols], sel
    # the stored tensors themselves (a detach() would be a new object without
    # the column statistics cached on it)
    return [_no_grad(c.values.data) for c in cols], None


def _no_grad(t: torch.Tensor) -> torch.Tensor:
    return t.detach() if t.requires_grad else t


def _is_catalog_column(cols: Sequence[EncodedTensor]) -> bool:
    """The side's columns are stored tensors (not lazy views): their range is
    worth a (cached) statistic."""
    return all(c.values._t is not None for c in cols)


def _gather_side(cols: Sequence[EncodedTensor], bases, rowmap, rows: torch.Tensor,
                 stats: bool = False):
    """Output columns of one join side: its (base) columns gathered at
    ``rows`` (through ``rowmap`` for a compacted side).  Outputs carry their
    base column's range statistic (computed once when ``stats``: the base is
    a catalog column), so a later join on them can run dense."""
    if not cols:
        return []
    if any(onehot_payload(c.values) is not None for c in cols):
        return [take_rows(c, rows if rowmap is None else gather_rows_raw(rowmap, rows))
                for c in cols]
    src = rows if rowmap is None else gather_rows_raw(rowmap, rows)
    outs = gather_many([b.contiguous() for b in bases], src)
    for o, b in zip(outs, bases):
        _inherit_range(o, b, compute=stats)
    with trusted():
        return [EncodedTensor(Tensor(o), c.encoding) for o, c in zip(outs, cols)]


def equi_join(left: Sequence[EncodedTensor], right: Sequence[EncodedTensor], left_key: int,
              right_key: int, left_out: Optional[Sequence[int]] = None,
              right_out: Optional[Sequence[int]] = None) -> list[EncodedTensor]:
    """Inner join ``left.left_key = right.right_key``; returns left columns then
    right columns, rows ordered by left row then ascending right row.  Keys
    must be plain int64 columns (dictionary codes from different dictionaries
    are not comparable).  Filtered (lazy) inputs are joined without
    materialising the filtered relations: only the key columns are gathered
    before the join, every output column is gathered once from its base.
    ``left_out`` / ``right_out`` (default: all) list the columns to return --
    a projection pushed into the join: the others are never gathered."""
    for side, cols, k in (("left", left, left_key), ("right", right, right_key)):
        col = cols[k]
        if col.is_pe() or col.is_dictionary() or col.values.dtype != "int64" or col.values.ndim != 1:
            raise KernelError(f"{side} join key must be a plain int64 column")
    lo = list(range(len(left))) if left_out is None else list(left_out)
    ro = list(range(len(right))) if right_out is None else list(right_out)
    for side, cols, out in (("left", left, lo), ("right", right, ro)):
        if any(not 0 <= i < len(cols) for i in out):
            raise KernelError(f"{side} output column index out of range")
    if active_tape() is not None:
        pi, bi = join_indices(left[left_key].values, right[right_key].values)
        return [take_rows(left[i], pi) for i in lo] + [take_rows(right[i], bi) for i in ro]
    group = current_group()
    if is_sharded(group):
        out = _equi_join_sharded(left, right, left_key, right_key, group)
        return [out[i] for i in lo] + [out[len(left) + i] for i in ro]
    if not ro:  # nothing from the right side: a semi-join, kept lazy when it can be
        semi = _semi_join_lazy(left, right, left_key, right_key, lo)
        if semi is not None:
            return semi
    lb, lsel = _side_sources(left)
    rb, rsel = _side_sources(right)
    # a filtered side whose key is a base column joins straight from the base
    # columns (its predicates run inside the join passes, row ids are base
    # ids); otherwise the side is compacted first
    lmap = rmap = None
    lkey_direct = lsel is not None and lb[left_key].dim() == 1
    rkey_direct = rsel is not None and rb[right_key].dim() == 1
    if not lkey_direct:
        lmap = lsel.indices() if lsel is not None else None
    lkey = lb[left_key] if lmap is None else gather_rows_raw(lb[left_key], lmap)
    # the build key's range (a column statistic) enables the dense-range join;
    # a semi-join (no right column returned) needs no build rows
    brange = column_range(rb[right_key], compute=rsel is not None or _is_catalog_column(right))
    need_rows = bool(ro)
    pairs = None
    if rkey_direct:
        pairs = join_indices(lkey, rb[right_key], probe_sel=lsel if lkey_direct else None,
                             build_sel=rsel, build_range=brange, need_build_rows=need_rows)
    if pairs is None:  # unfiltered build side, or a filtered one with repeated keys
        rmap = rsel.indices() if rsel is not None else None
        rkey = rb[right_key] if rmap is None else gather_rows_raw(rb[right_key], rmap)
        pairs = join_indices(lkey, rkey, probe_sel=lsel if lkey_direct else None,
                             build_range=brange if rmap is None else None,
                             need_build_rows=need_rows)
    pi, bi = pairs
    lcols, rcols = [left[i] for i in lo], [right[i] for i in ro]
    if lcols and rcols and len(lo) + len(ro) <= 16 and bi is not None and not any(
            onehot_payload(c.values) is not None for c in lcols + rcols):
        return _gather_sides(lcols, [lb[i] for i in lo], lmap, pi, lsel is not None,
                             rcols, [rb[i] for i in ro], rmap, bi, rsel is not None)
    return (_gather_side(lcols, [lb[i] for i in lo], lmap, pi, stats=lsel is not None)
            + _gather_side(rcols, [rb[i] for i in ro], rmap, bi, stats=rsel is not None))


def _gather_sides(lcols, lbases, lmap, prows, lstats, rcols, rbases, rmap, brows, rstats):
    """Both sides' output columns of a join in one launch (tdp_gather_rows2):
    left columns at the probe rows, right columns at the build rows."""
    lsrc = prows if lmap is None else gather_rows_raw(lmap, prows)
    rsrc = brows if rmap is None else gather_rows_raw(rmap, brows)
    bases = [b.contiguous() for b in list(lbases) + list(rbases)]
    nat.require_cuda(lsrc, rsrc, *bases)
    m = int(lsrc.numel())
    outs = [torch.empty((m,) + tuple(b.shape[1:]), dtype=b.dtype, device=b.device) for b in bases]
    if m:
        dst = (c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        nat.call("tdp_gather_rows2", nat.columns(bases), len(bases), len(lbases), nat.ptr(lsrc),
                 nat.ptr(rsrc), m, dst, nat.stream())
    for k, (o, b) in enumerate(zip(outs, bases)):
        _inherit_range(o, b, compute=lstats if k < len(lbases) else rstats)
    cols = list(lcols) + list(rcols)
    with trusted():
        return [EncodedTensor(Tensor(o), c.encoding) for o, c in zip(outs, cols)]


def _semi_join_lazy(left, right, left_key: int, right_key: int, lo: list):
    """``left`` joined with ``right`` when no right column is returned and the
    right keys are unique: exactly the left rows whose key is among the right
    keys, in left row order.  It stays lazy -- the left selection refined by a
    membership predicate on a bitmap of the right keys (TDP_CMP_BITMAP, one
    bit per value of the right key's range) -- so no pairs are formed and a
    later consumer (another join's build, a fused aggregate) evaluates it in
    its own pass.  None (the caller runs the pair join) when the left side is
    not one row space of base columns, the right key has no usable range
    statistic, or a right key repeats (one host read of the build flags)."""
    space = _row_space(left)
    if space is None:
        return None
    lsel, n_left = space
    kv = left[left_key].values
    if kv._t is not None:
        lbase = kv._t
    elif isinstance(kv._lazy, LazyValue) and kv._lazy.expr.op == "col":
        lbase = kv._lazy.expr.col
    else:
        return None
    rb, rsel = _side_sources(right)
    if rsel is None and not _is_catalog_column(right):
        return None
    bk = rb[right_key]
    if bk.dim() != 1 or bk.dtype != torch.int64 or lbase.dtype != torch.int64:
        return None
    n_build = int(bk.numel())
    dense = _dense_range(column_range(bk), n_build)
    if dense is None or n_build == 0:
        return None
    nat.require_cuda(bk, lbase)
    lo_key, span = dense
    dev = bk.device
    bits = torch.empty((span + 31) // 32, dtype=torch.int32, device=dev)
    flags = torch.empty(2, dtype=torch.int32, device=dev)
    if rsel is not None and rsel.preds:
        if rsel.n != n_build:
            raise KernelError("build selection and key column disagree on row count")
        prog = Program()
        preds, npreds = prog.predicates(rsel)
        nat.require_cuda(*prog.cols)
        bc, nbc = prog.native_columns(), len(prog.cols)
    else:
        bc, nbc, preds, npreds = nat.columns([]), 0, nat.struct_array(nat.Predicate, []), 0
    nat.call("tdp_join_dense_bitmap", nat.ptr(bk.contiguous()), n_build, bc, nbc, preds, npreds,
             lo_key, span, nat.ptr(bits), nat.ptr(flags), nat.stream())
    if any(read_ints(flags)):  # a repeated (or out-of-statistic) right key
        return None
    member = Pred(lbase, "=", nat.CMP_BITMAP, lo_key, float(span), aux=bits)
    device = _device_of([as_expr(c.values)[0] for c in left], lsel)
    new_sel = lsel.refine([member]) if lsel is not None else Selection(n_left, [member], device)
    out = []
    for i in lo:
        c = left[i]
        v = c.values
        expr = Expr.column(v._t) if v._t is not None else v._lazy.expr
        with trusted():
            out.append(EncodedTensor(Tensor(LazyValue(expr, new_sel, valid_for=c.encoding)),
                                     c.encoding))
    return out


def _repartition(cols: Sequence[EncodedTensor], key_index: int, group) -> list[EncodedTensor]:
    """Rows of one (row-sharded) relation moved to the rank that owns their
    join key (key_destination), by an NCCL all-to-all; encodings kept."""
    data = []
    for c in cols:
        if c.is_pe() or c.values.ndim != 1:
            raise KernelError("a sharded join moves scalar columns only")
        t = c.values.data.detach()
        data.append(t.to(torch.int64) if t.dtype == torch.bool else t.contiguous())
    world = world_size(group)
    dest = key_destination([data[key_index]], world)
    n = int(dest.numel())
    order = stable_order(plain(Tensor(dest)))
    send_counts, _ = _groupby_codes(dest, world, [], [], n, dest.device)
    moved = exchange_rows(gather_many(data, order), send_counts, group)
    out = []
    with trusted():
        for c, t, orig in zip(cols, moved, data):
            if c.values.dtype == "bool":
                t = t.to(torch.bool)
            out.append(EncodedTensor(Tensor(t), c.encoding))
    return out


def _equi_join_sharded(left, right, left_key: int, right_key: int, group) -> list[EncodedTensor]:
    """Equi-join of two row-sharded relations: both sides are
    repartitioned by key with an all-to-all, so every key's rows meet on one
    rank, then joined locally.  The result is again row-sharded (each rank
    holds the pairs of the keys it owns); its row order is by rank of
    arrival, as the join's order is not part of its contract."""
    lp = _repartition(left, left_key, group)
    rp = _repartition(right, right_key, group)
    pi, bi = join_indices(lp[left_key].values, rp[right_key].values)
    return [take_rows(c, pi) for c in lp] + [take_rows(c, bi) for c in rp]


# ---------------------------------------------------------------------------
# UDF / TVF registry (tq/kernels.py:288-369)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class UdfEntry:
    """A registered function: declared outputs, arity, body and parameters."""

    name: str
    output_schema: tuple[tuple[str, ColumnType], ...]
    arity: int
    body: Callable[..., tuple[EncodedTensor, ...]]
    params: tuple[Parameter, ...] = ()
    pe_outputs: bool = True


def _row_keys(outputs: Sequence[EncodedTensor]) -> set:
    """Row counts of outputs, compared symbolically for lazy views of one selection."""
    keys = set()
    for o in outputs:
        v = o.values
        if v._t is None and isinstance(v._lazy, LazyValue) and v._lazy.sel is not None \
                and v._lazy.sel._count is None:
            keys.add(("sel", id(v._lazy.sel)))
        else:
            keys.add(o.row_count)
    return keys


class UdfRegistry:
    """Insertion-ordered function registry; registrations are exclusive."""

    def __init__(self):
        self._entries: dict[str, UdfEntry] = {}

    def register(self, entry: UdfEntry) -> UdfEntry:
        if entry.name in self._entries:
            raise KernelError(f"function {entry.name!r} is already registered")
        seen = set()
        for p in entry.params:
            if p.name in seen:
                raise KernelError(f"duplicate parameter name {p.name!r} in {entry.name!r}")
            seen.add(p.name)
        self._entries[entry.name] = entry
        return entry

    def lookup(self, name: str) -> Optional[UdfEntry]:
        return self._entries.get(name)

    def names(self) -> list[str]:
        return list(self._entries)

    def entries(self) -> list[UdfEntry]:
        return list(self._entries.values())

    def invoke(self, name: str, inputs: Sequence[EncodedTensor]) -> tuple[EncodedTensor, ...]:
        entry = self._entries.get(name)
        if entry is None:
            raise KernelError(f"unknown function {name!r}")
        if len(inputs) != entry.arity:
            raise KernelError(f"function {name!r} takes {entry.arity} argument(s), got {len(inputs)}")
        outputs = entry.body(*inputs)
        if isinstance(outputs, EncodedTensor):
            outputs = (outputs,)
        outputs = tuple(outputs)
        self._validate_outputs(entry, outputs)
        return outputs

    @staticmethod
    def _validate_outputs(entry: UdfEntry, outputs: tuple[EncodedTensor, ...]) -> None:
        declared = entry.output_schema
        if len(outputs) != len(declared):
            raise KernelError(
                f"function {entry.name!r} declared {len(declared)} output column(s), "
                f"returned {len(outputs)}"
            )
        rows = _row_keys(outputs)
        if len(rows) > 1:
            counts = sorted({o.row_count for o in outputs})
            if len(counts) > 1:
                raise KernelError(
                    f"function {entry.name!r} returned columns with differing row counts {counts}"
                )
        for (name, ctype), out in zip(declared, outputs):
            if ctype.kind == "tensor" and entry.pe_outputs:
                if not out.is_pe() or out.encoding.num_classes != ctype.dims[0]:
                    raise KernelError(
                        f"output {name!r} of {entry.name!r} must be PE over {ctype.dims[0]} classes"
                    )
            elif ctype.kind == "string":
                if not out.is_dictionary():
                    raise KernelError(f"output {name!r} of {entry.name!r} must be a string column")
            elif ctype.kind in ("int", "float"):
                if out.values.ndim != 1:
                    raise KernelError(f"output {name!r} of {entry.name!r} must be a scalar column")


def make_scoring_udf(name: str, weights: Tensor, scale: float = 1.0,
                     column: str = "Score") -> UdfEntry:
    """Generic scoring hook: rows -> plain float score, x . w / scale."""
    if weights.ndim != 1:
        raise KernelError("scoring weights must be a vector")
    d = int(weights.shape[0])

    def body(col: EncodedTensor) -> tuple[EncodedTensor, ...]:
        x = col.values
        if x.ndim != 2 or x.shape[1] != d:
            raise KernelError(f"scoring input must be [n, {d}]")
        from .tensor import matmul

        scores = mul(reshape(matmul(x, reshape(weights, (d, 1))), (x.shape[0],)),
                     tensor(1.0 / scale, dtype=x.dtype))
        return (plain(scores),)

    return UdfEntry(name, ((column, ColumnType("float")),), 1, body, (), pe_outputs=False)

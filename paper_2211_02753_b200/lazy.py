"""Late materialisation: lazy filter selections and elementwise expressions.

The reference executes one operator at a time and materialises every column
of every intermediate relation (tq/compiler.py:366-367; filter_exact compacts
all columns, tq/kernels.py:96-97).  Here a filter yields a :class:`Selection`
(the conjunction of its predicates over the base columns) and the relation's
columns become lazy references to base columns under that selection.  An
elementwise UDF body over such columns (add/sub/mul/div/neg/square/log/exp/
relu, tq/tensor.py:330-412) records a small expression DAG instead of
computing.  A consumer either

* materialises a value (``Tensor.data``): predicate pass + compaction + gather
  or the NVRTC-specialised projection kernel, or
* consumes the whole thing in one fused pass (group-by / global aggregate:
  ``tdp_scan_aggregate``), reading each base column once.

Results are identical to eager evaluation: predicates use the numpy NEP 50
comparison type resolved on the host, expressions use numpy's dtype promotion
and are evaluated without FMA contraction.
"""

from __future__ import annotations

import struct
import threading
import weakref
from ctypes import c_int32, c_void_p
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native as nat
from .hostread import SYNC_READS, read_int, record_value, replay_value
from . import autograd as _ag
from . import tensor as _T

INT64_MIN, INT64_MAX = -(2**63), 2**63 - 1

_LAZY_OPS = ("add", "sub", "mul", "div", "neg", "square", "log", "exp", "relu")
_OPCODE = {"add": nat.OP_ADD, "sub": nat.OP_SUB, "mul": nat.OP_MUL, "div": nat.OP_DIV,
           "neg": nat.OP_NEG, "square": nat.OP_SQUARE, "log": nat.OP_LOG, "exp": nat.OP_EXP,
           "relu": nat.OP_RELU}
_PROGRAM_DTYPES = ("int64", "float64", "float32")


# ---------------------------------------------------------------------------
# predicates (tq/kernels.py:54-84)
# ---------------------------------------------------------------------------

def resolve_predicate(col_dtype: str, op: str, literal) -> tuple[int, int, float]:
    """(compare kind, int literal, float literal) with numpy-2 promotion.

    ``np.result_type`` applies NEP 50: Python scalars are weak (a float32
    column compares against float32(literal), an int64 column against a
    Python float compares in float64), numpy scalars are strong.
    """
    if isinstance(literal, (bool, np.bool_)):
        literal = int(literal)
    if isinstance(literal, int) and not isinstance(literal, np.integer):
        if col_dtype in ("int64", "bool") and not INT64_MIN <= literal <= INT64_MAX:
            if col_dtype == "bool":
                raise OverflowError("Python int too large to convert to C long")
            above = literal > INT64_MAX
            always = {"=": False, "<>": True, "<": above, "<=": above, ">": not above,
                      ">=": not above}[op]
            return (nat.CMP_ALL if always else nat.CMP_NONE), 0, 0.0
    rt = np.result_type(np.empty(0, dtype=col_dtype), literal)
    if rt.kind in "iub":
        return nat.CMP_I64, int(literal), 0.0
    if rt == np.float32:
        return nat.CMP_F32, 0, float(np.float32(literal))
    return nat.CMP_F64, 0, float(np.float64(literal))


class Pred:
    """One resolved comparison on a base column.  ``aux`` is the operand
    tensor of a semi-join membership test (CMP_BITMAP: the bitmap of the
    right side's keys, lit_i = lowest key, lit_f = key range)."""

    __slots__ = ("col", "op", "cmp", "lit_i", "lit_f", "aux")

    def __init__(self, col: Optional[torch.Tensor], op: str, cmp: int, lit_i: int, lit_f: float,
                 aux: Optional[torch.Tensor] = None):
        self.col = col
        self.op = op
        self.cmp = cmp
        self.lit_i = lit_i
        self.lit_f = lit_f
        self.aux = aux


def native_predicates(preds: Sequence[Pred], col_index: dict[int, int]):
    arr = (nat.Predicate * max(1, len(preds)))()
    for k, p in enumerate(preds):
        c = col_index[id(p.col)] if p.col is not None else 0
        aux = col_index[id(p.aux)] if p.aux is not None else 0
        arr[k] = nat.Predicate(c, nat.CMP_OPS[p.op], p.cmp, aux, p.lit_i, p.lit_f)
    return arr


class Selection:
    """Rows of one base row space passing a conjunction of predicates."""

    __slots__ = ("n", "preds", "device", "_idx", "_count_dev", "_count")

    def __init__(self, n: int, preds: Sequence[Pred], device: torch.device):
        self.n = int(n)
        self.preds = tuple(preds)
        self.device = device
        self._idx: Optional[torch.Tensor] = None
        self._count_dev: Optional[torch.Tensor] = None
        self._count: Optional[int] = None

    def refine(self, preds: Sequence[Pred]) -> "Selection":
        return Selection(self.n, self.preds + tuple(preds), self.device)

    def base_columns(self) -> list[torch.Tensor]:
        """Predicate operands: the base columns and any semi-join bitmaps."""
        cols, seen = [], set()
        for p in self.preds:
            for t in (p.col, p.aux):
                if t is not None and id(t) not in seen:
                    seen.add(id(t))
                    cols.append(t)
        return cols

    def _run(self) -> None:
        cols = self.base_columns()
        if not cols:
            # every predicate is a constant (absent dictionary literal / range)
            keep_all = all(p.cmp == nat.CMP_ALL for p in self.preds)
            m = self.n if keep_all else 0
            self._idx = torch.arange(m, dtype=torch.int64, device=self.device)
            self._count = m
            return
        nat.require_cuda(*cols)
        index = {id(c): i for i, c in enumerate(cols)}
        out_idx = torch.empty(max(self.n, 1), dtype=torch.int64, device=self.device)
        count = torch.empty(1, dtype=torch.int64, device=self.device)
        ws = nat.workspace(nat.load().tdp_filter_workspace(self.n), self.device)
        nat.call("tdp_filter_select", nat.columns(cols), len(cols),
                 native_predicates(self.preds, index), len(self.preds), self.n,
                 nat.ptr(out_idx), nat.ptr(count), nat.ptr(ws), ws.numel(), nat.stream())
        self._count_dev = count
        self._count = read_int(count)
        self._idx = out_idx[: self._count]

    def indices(self) -> torch.Tensor:
        if self._idx is None:
            self._run()
        return self._idx

    def count(self) -> int:
        if self._count is None:
            self._run()
        return self._count


# ---------------------------------------------------------------------------
# expressions
# ---------------------------------------------------------------------------

class Expr:
    """Node of an elementwise expression over base columns."""

    __slots__ = ("op", "dtype", "args", "col", "value")

    def __init__(self, op: str, dtype: str, args: tuple = (), col: Optional[torch.Tensor] = None,
                 value=None):
        self.op = op
        self.dtype = dtype
        self.args = args
        self.col = col
        self.value = value

    @staticmethod
    def column(t: torch.Tensor) -> "Expr":
        return Expr("col", _T.dtype_name(t), col=t)

    @staticmethod
    def const(value, dtype: str) -> "Expr":
        return Expr("const", dtype, value=value)

    def cast(self, dtype: str) -> "Expr":
        return self if dtype == self.dtype else Expr("cast", dtype, (self,))


NARROW_INTS = ("int32", "int16", "int8", "uint8")


def set_value_range(t: torch.Tensor, lo: int, hi: int) -> None:
    """Record that every value of the (immutable, narrow integer) stored column
    ``t`` lies in [lo, hi] -- measured at ingestion by compact storage.  The
    fused scan uses it to bound exact integer sums (TDP_OP_LOAD range hint)."""
    t._tdp_range = (int(lo), int(hi))


def value_range(t: torch.Tensor) -> Optional[tuple[int, int]]:
    r = getattr(t, "_tdp_range", None)
    if r is None or t.dtype not in (torch.int32, torch.int16, torch.int8, torch.uint8):
        return None
    return r


def compact_source(e: Expr) -> Optional[tuple[torch.Tensor, int]]:
    """(stored narrow column, decimal divisor or 0) when ``e`` decodes a
    compact column (compact.py): ``cast(col)`` to int64, or
    ``cast(col) / const`` to float64."""
    if e.op == "cast" and e.dtype == "int64" and e.args[0].op == "col" \
            and e.args[0].dtype in NARROW_INTS:
        return e.args[0].col, 0
    if e.op == "decimal" and e.args[0].op == "cast" and e.args[0].args[0].op == "col" \
            and e.args[0].args[0].dtype in NARROW_INTS:
        return e.args[0].args[0].col, int(e.value)
    if e.op == "cast" and e.dtype == "float64" and e.args[0].op == "cast" \
            and e.args[0].dtype == "int64" and e.args[0].args[0].op == "col" \
            and e.args[0].args[0].dtype in NARROW_INTS:
        return e.args[0].args[0].col, 1
    return None


def decimal_predicates(op: str, lit: float, divisor: int) -> list[tuple[str, int, int]]:
    """``value <op> lit`` on a column stored as integers c with value =
    RN(c / divisor) (compact.py verifies it for every stored row), as
    conjunctions of int64 comparisons on c: [(op, compare kind, int literal)].

    RN(c / d) is non-decreasing in c, so {c : RN(c/d) >= lit} = {c >= t} with
    t found by bisection in exact arithmetic (Python int / int is correctly
    rounded).  A NaN literal matches nothing except under <>."""
    if lit != lit:
        return [(op, nat.CMP_ALL if op == "<>" else nat.CMP_NONE, 0)]
    lo_b, hi_b = -(2**62), 2**62

    def first(pred) -> int:  # smallest c in [lo_b, hi_b] with pred(c), else hi_b + 1
        lo, hi = lo_b, hi_b + 1
        while lo < hi:
            mid = (lo + hi) // 2
            if pred(mid):
                hi = mid
            else:
                lo = mid + 1
        return lo

    t_ge = first(lambda c: c / divisor >= lit)
    t_gt = first(lambda c: c / divisor > lit)
    if op == ">=":
        return [(">=", nat.CMP_I64, t_ge)]
    if op == ">":
        return [(">=", nat.CMP_I64, t_gt)]
    if op == "<":
        return [("<", nat.CMP_I64, t_ge)]
    if op == "<=":
        return [("<", nat.CMP_I64, t_gt)]
    if op == "=":
        if t_gt == t_ge:
            return [("=", nat.CMP_NONE, 0)]
        if t_gt == t_ge + 1:
            return [("=", nat.CMP_I64, t_ge)]
        return [(">=", nat.CMP_I64, t_ge), ("<", nat.CMP_I64, t_gt)]
    # "<>"
    if t_gt == t_ge:
        return [("<>", nat.CMP_ALL, 0)]
    if t_gt == t_ge + 1:
        return [("<>", nat.CMP_I64, t_ge)]
    return [("<>", nat.CMP_DEC, divisor)]  # several stored values decode to lit


class LazyValue:
    """An unmaterialised column: ``expr`` evaluated on the rows of ``sel``."""

    __slots__ = ("expr", "sel", "dtype", "valid_for")

    def __init__(self, expr: Expr, sel: Optional[Selection], valid_for=None):
        self.expr = expr
        self.sel = sel
        self.dtype = expr.dtype
        self.valid_for = valid_for  # encoding the values are known to satisfy

    @property
    def ndim(self) -> int:
        return self.expr.col.dim() if self.expr.op == "col" else 1

    def rows(self) -> int:
        if self.sel is not None:
            return self.sel.count()
        return base_rows(self.expr)

    def shape(self) -> tuple:
        tail = tuple(self.expr.col.shape[1:]) if self.expr.op == "col" else ()
        return (self.rows(),) + tail

    def materialize(self) -> torch.Tensor:
        e = self.expr
        if e.op == "col":
            if self.sel is None:
                return e.col
            return _ag.gather_rows_raw(e.col, self.sel.indices())
        return project([e], self.sel)[0]


def base_rows(e: Expr) -> int:
    if e.op == "col":
        return int(e.col.shape[0])
    for a in e.args:
        n = base_rows(a)
        if n >= 0:
            return n
    return -1


def lazy_view(t: torch.Tensor, sel: Selection, valid_for=None) -> LazyValue:
    return LazyValue(Expr.column(t), sel, valid_for)


def as_expr(value) -> tuple[Expr, Optional[Selection]]:
    """(expression, selection) of a Tensor (lazy or materialised) or torch tensor."""
    if isinstance(value, _T.Tensor):
        if value._t is None and isinstance(value._lazy, LazyValue):
            return value._lazy.expr, value._lazy.sel
        value = value.data
    return Expr.column(value.contiguous()), None


def _lazy_operand(t, rdt: str):
    """Expr and selection for ``t`` as an operand of a lazy op, or None."""
    if not isinstance(t, _T.Tensor):
        return None
    if t._t is None:
        lv = t._lazy
        if not isinstance(lv, LazyValue) or lv.ndim != 1:
            return None
        return lv.expr.cast(rdt), lv.sel, True
    if t._t.dim() == 0:
        if t.node is not None or t._t.requires_grad:
            return None
        v = t._scalar if t._scalar is not None else t._t.item()
        return Expr.const(v, t.dtype).cast(rdt), None, False
    return None


def try_lazy_binary(op: str, a, b, rdt: str):
    if op not in _LAZY_OPS or rdt not in _PROGRAM_DTYPES:
        return None
    la = _lazy_operand(a, rdt)
    lb = _lazy_operand(b, rdt)
    if la is None or lb is None or not (la[2] or lb[2]):
        return None
    sa, sb = la[1], lb[1]
    if sa is not None and sb is not None and sa is not sb:
        return None
    sel = sa if sa is not None else sb
    if op == "div" and rdt == "int64":
        return None
    return _T.Tensor(LazyValue(Expr(op, rdt, (la[0], lb[0])), sel))


def try_lazy_unary(op: str, a, rdt: str):
    if op not in _LAZY_OPS or rdt not in _PROGRAM_DTYPES:
        return None
    la = _lazy_operand(a, rdt)
    if la is None or not la[2]:
        return None
    if op in ("log", "exp", "relu") and rdt == "int64":
        return None
    return _T.Tensor(LazyValue(Expr(op, rdt, (la[0],)), la[1]))


# ---------------------------------------------------------------------------
# program compilation (Expr DAG -> tdp_instr SSA program)
# ---------------------------------------------------------------------------

_DT = {"int64": nat.I64, "float64": nat.F64, "float32": nat.F32}


class Program:
    """SSA program over a deduplicated list of base columns."""

    def __init__(self):
        self.cols: list[torch.Tensor] = []
        self._col_index: dict[int, int] = {}
        self.instrs: list[nat.Instr] = []
        self._memo: dict[tuple, int] = {}

    def col_index(self, t: torch.Tensor) -> int:
        k = id(t)
        if k not in self._col_index:
            self._col_index[k] = len(self.cols)
            self.cols.append(t)
        return self._col_index[k]

    def _emit(self, key: tuple, ins: nat.Instr) -> int:
        v = self._memo.get(key)
        if v is None:
            v = len(self.instrs)
            self.instrs.append(ins)
            self._memo[key] = v
        return v

    def value(self, e: Expr) -> int:
        if e.op == "col":
            if e.col.dim() != 1:
                raise ValueError("expression columns must be 1-d")
            c = self.col_index(e.col)
            load_dt = {"int64": "int64", "bool": "int64", "float64": "float64",
                       "float32": "float32", "int32": "int64", "int16": "int64",
                       "int8": "int64", "uint8": "int64"}[e.dtype]
            rng = value_range(e.col) if load_dt == "int64" else None
            if rng is not None:  # promised [lo, hi]: lets sums run as exact packed integers
                ins = nat.Instr(nat.OP_LOAD, _DT[load_dt], c, 1, rng[0], float(rng[1]))
            else:
                ins = nat.Instr(nat.OP_LOAD, _DT[load_dt], c, 0, 0, 0.0)
            return self._emit(("load", c), ins)
        if e.op == "const":
            dt = e.dtype if e.dtype in _DT else "int64"
            if dt == "int64":
                iv = int(e.value)
                return self._emit(("ci", iv), nat.Instr(nat.OP_CONST, nat.I64, 0, 0, iv, 0.0))
            fv = float(e.value)
            bits = struct.pack("<d", fv)
            return self._emit(("cf", dt, bits), nat.Instr(nat.OP_CONST, _DT[dt], 0, 0, 0, fv))
        if e.op == "decimal":  # compact float64 column: stored integer / divisor
            a = self.value(e.args[0])
            d = float(e.value)
            inv_bits = struct.unpack("<q", struct.pack("<d", 1.0 / d))[0]
            return self._emit(("dec", a, d), nat.Instr(nat.OP_DECIMAL, nat.F64, a, 0, inv_bits, d))
        if e.op == "cast":
            a = self.value(e.args[0])
            src = self.instrs[a].dtype
            if src == _DT[e.dtype]:
                return a
            return self._emit(("cast", e.dtype, a), nat.Instr(nat.OP_CAST, _DT[e.dtype], a, 0, 0, 0.0))
        args = [self.value(x) for x in e.args]
        dt = _DT[e.dtype]
        for x in args:
            if self.instrs[x].dtype != dt:
                raise ValueError("operand dtype mismatch in lazy expression")
        a = args[0]
        b = args[1] if len(args) > 1 else 0
        return self._emit((e.op, e.dtype, a, b), nat.Instr(_OPCODE[e.op], dt, a, b, 0, 0.0))

    def predicates(self, sel: Optional[Selection]):
        preds = sel.preds if sel is not None else ()
        for p in preds:
            if p.col is not None:
                self.col_index(p.col)
            if p.aux is not None:
                self.col_index(p.aux)
        return native_predicates(preds, self._col_index), len(preds)

    def native_columns(self):
        return nat.columns(self.cols)

    def native_instrs(self):
        return nat.struct_array(nat.Instr, self.instrs)


def project(exprs: Sequence[Expr], sel: Optional[Selection]) -> list[torch.Tensor]:
    """Materialise expressions on the selected rows (tdp_scan_project)."""
    prog = Program()
    outs = [prog.value(e) for e in exprs]
    preds, npreds = prog.predicates(sel)
    n = base_rows(exprs[0]) if exprs else 0
    if n < 0 and sel is not None:
        n = sel.n
    nat.require_cuda(*prog.cols)
    device = prog.cols[0].device if prog.cols else (sel.device if sel else torch.device("cuda"))
    m = sel.count() if sel is not None else n
    results = [torch.empty(m, dtype=_T.torch_dtype(e.dtype), device=device) for e in exprs]
    if m == 0 or not prog.cols:
        if not prog.cols:  # constant expression
            return [torch.full((m,), float(e.value) if e.dtype != "int64" else int(e.value),
                               dtype=_T.torch_dtype(e.dtype), device=device) for e in exprs]
        return results
    count = torch.empty(1, dtype=torch.int64, device=device)
    ws = nat.workspace(nat.load().tdp_filter_workspace(n), device)
    out_idx = (c_int32 * len(outs))(*outs)
    out_ptrs = (c_void_p * len(results))(*[r.data_ptr() for r in results])
    nat.call("tdp_scan_project", prog.native_columns(), len(prog.cols), n, preds, npreds,
             prog.native_instrs(), len(prog.instrs), out_idx, len(outs), out_ptrs,
             nat.ptr(count), nat.ptr(ws), ws.numel(), nat.stream())
    return results


# ---------------------------------------------------------------------------
# device-resident row counts (results whose length the host has not read yet)
# ---------------------------------------------------------------------------


_CAPTURE = threading.local()


class capturing:
    """Context of a CUDA-graph capture of a query (compiler.py): device
    counts stay on the device (no host copy or event inside the graph)."""

    def __enter__(self):
        _CAPTURE.on = True
        return self

    def __exit__(self, *exc):
        _CAPTURE.on = False


def is_capturing() -> bool:
    return getattr(_CAPTURE, "on", False)


class DeferredCount:
    """A row count produced by a kernel, left on the device until first
    access: an event is recorded after the producing launch, and ``value()``
    waits for it and reads the count then.  A query whose result stays on the
    device neither blocks the launching thread nor queues a device-to-host
    copy behind its kernels (each such copy in a replayed step's stream costs
    a copy-engine round trip: compact Q1 step 170 -> 159 us without it)."""

    __slots__ = ("_event", "_value", "dev", "_template", "__weakref__")

    def __init__(self, dev: torch.Tensor):
        self._value: Optional[int] = None
        self.dev = dev
        self._template = is_capturing()  # a graph template: the replay makes a real one
        self._event = None
        if not self._template:
            self._event = torch.cuda.Event()
            self._event.record()

    def value(self) -> int:
        if self._value is None:
            if self._template:
                v = replay_value(self.dev)  # a capture sized from a recorded run
                if v is None:
                    raise RuntimeError("row count of a CUDA-graph template read during capture")
                self._value = v
                return v
            SYNC_READS[0] += 1
            self._event.synchronize()  # the producing stream's count is final
            self._value = int(self.dev.reshape(-1)[0].item())
            record_value(self._value)
            self._event = None
            self.dev = None
        return self._value


class PrefixRows:
    """Lazy payload: the first ``count`` rows of ``full`` (a padded result
    buffer written by a kernel whose row count is a :class:`DeferredCount`)."""

    __slots__ = ("full", "count", "dtype")

    def __init__(self, full: torch.Tensor, count: DeferredCount):
        self.full = full
        self.count = count
        self.dtype = _T.dtype_name(full)

    @property
    def ndim(self) -> int:
        return self.full.dim()

    def shape(self) -> tuple:
        return (self.count.value(),) + tuple(self.full.shape[1:])

    def materialize(self) -> torch.Tensor:
        return self.full[: self.count.value()]


def deferred_rows(t) -> Optional[DeferredCount]:
    """The DeferredCount of an unresolved PrefixRows tensor, else None."""
    if isinstance(t, _T.Tensor) and t._t is None and isinstance(t._lazy, PrefixRows) \
            and t._lazy.count._value is None:
        return t._lazy.count
    return None


class SelectionRows:
    """Row count of a filtered relation that has not been evaluated yet: a
    result table over lazy views reads it (running the filter) only when its
    ``row_count`` or a column's data is first needed."""

    __slots__ = ("sel",)

    def __init__(self, sel: Selection):
        self.sel = sel

    def value(self) -> int:
        return self.sel.count()


def deferred_selection(columns) -> Optional[Selection]:
    """The common unevaluated Selection of columns that are all lazy views of
    it (values of EncodedTensors), else None."""
    sel = None
    for c in columns:
        t = c.values
        if not (isinstance(t, _T.Tensor) and t._t is None and isinstance(t._lazy, LazyValue)):
            return None
        s = t._lazy.sel
        if s is None or s._count is not None or (sel is not None and s is not sel):
            return None
        sel = s
    return sel

"""Compact column storage (narrow encodings at ingestion).

The reference stores every column at 8 bytes per value: int64 dates and
dictionary codes, float64 prices (tq/storage.py:190-249, tq/encodings.py:88).
A scan-bound query moves those 8 bytes per column per row, over HBM in the
fused pass and over PCIe when the table starts in host memory.  Here a column
can be *stored* narrow while keeping its logical type, values and encoding:

* int64 column / dictionary codes -> int8 / uint8 / int16 / int32 when every
  value fits (dates are day numbers < 32768: int16; dictionary codes of a
  <= 256-entry dictionary: uint8);
* float64 column -> scaled integers ``c`` with ``value == c / 10**s`` *bit for
  bit* (checked on every row at ingestion; TPC-H money and rates are 2-decimal
  numbers), stored in the narrowest integer type holding ``c``.

A compact column is a lazy expression over its stored tensor (lazy.py):
``cast(stored)`` for integers, ``decimal(cast(stored), 10**s)`` for decimals
(TDP_OP_DECIMAL: the correctly rounded quotient from one multiply and two
FMAs -- no divide in the scan loop; ingestion checks it bit for bit).  The
fused scan decodes in registers; a filter on a decimal column becomes an int64
comparison on the stored integers (RN(c / 10**s) is monotone in c, so
``value >= lit`` is ``c >= t`` for an exactly computed t,
lazy.decimal_predicates); any other consumer materialises the decoded column
through the projection kernel.
Results are therefore identical to the uncompacted table: the decoded values
are the original float64 / int64 values.  A column that does not round-trip
(non-decimal floats, -0.0, NaN, out-of-range integers) stays as it is.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from .encodings import EncodedTensor, trusted
from .lazy import Expr, LazyValue, compact_source, project, set_value_range
from .storage import Table, table_from_columns
from .tensor import Tensor

_INT_TYPES = ((torch.int8, -(2**7), 2**7 - 1), (torch.int16, -(2**15), 2**15 - 1),
              (torch.int32, -(2**31), 2**31 - 1))
_NARROW_NAME = {torch.int8: "int8", torch.int16: "int16", torch.int32: "int32",
                torch.uint8: "uint8", torch.int64: "int64"}
DECIMAL_SCALES = (1, 10, 100, 1000, 10000)


@dataclass(frozen=True)
class CompactSpec:
    """How one column is stored: torch dtype of the stored values and the
    decimal divisor (0 for integer columns)."""

    stored: torch.dtype
    divisor: int = 0


def _int_type(lo: int, hi: int, unsigned_ok: bool) -> Optional[torch.dtype]:
    if unsigned_ok and lo >= 0 and hi <= 255:
        return torch.uint8
    for dt, a, b in _INT_TYPES:
        if a <= lo and hi <= b:
            return dt
    return None


def decode_expr(stored: torch.Tensor, divisor: int) -> Expr:
    """Expression giving the logical values of a stored compact column:
    ``cast`` to int64, then for decimals the divide-free correctly rounded
    quotient by ``divisor`` (TDP_OP_DECIMAL)."""
    col = Expr("cast", "int64", (Expr("col", _NARROW_NAME[stored.dtype], col=stored),))
    if divisor == 1:  # integer-valued floats: the conversion is exact
        return Expr("cast", "float64", (col,))
    if divisor:
        return Expr("decimal", "float64", (col,), value=int(divisor))
    return col


def from_stored(stored: torch.Tensor, spec: CompactSpec, like: EncodedTensor) -> EncodedTensor:
    """Compact column over already-narrow stored values (e.g. just copied from
    host memory), with the encoding of ``like``."""
    if stored.dtype != spec.stored or stored.dim() != 1:
        raise ValueError(f"stored column must be 1-d {spec.stored}, got {stored.dtype}")
    lv = LazyValue(decode_expr(stored.contiguous(), spec.divisor), None, valid_for=like.encoding)
    with trusted():
        return EncodedTensor(Tensor(lv), like.encoding)


def plan_column(col: EncodedTensor) -> Optional[tuple[CompactSpec, torch.Tensor]]:
    """(spec, stored values) for a lossless narrow form of ``col``, or None."""
    v = col.values
    if v.ndim != 1 or col.is_pe() or (v._t is None and not isinstance(v._lazy, LazyValue)):
        return None
    if v._t is None and compact_source(v._lazy.expr) is not None:
        return None  # already compact
    t = v.data
    n = int(t.shape[0])
    if t.dtype == torch.int64:
        if n == 0:
            return None
        lo, hi = (int(x) for x in torch.aminmax(t))
        dt = _int_type(lo, hi, unsigned_ok=col.is_dictionary())
        if dt is None:
            return None
        stored = t.to(dt)
        set_value_range(stored, lo, hi)
        return CompactSpec(dt), stored
    if t.dtype != torch.float64 or n == 0:
        return None
    # exact decimal test on the host (numpy division is correctly rounded),
    # then the device decode itself is checked bit for bit
    host = t.cpu().numpy()
    bits = host.view(np.int64)
    with np.errstate(all="ignore"):
        for s in DECIMAL_SCALES:
            c = np.rint(host * s)
            if not np.isfinite(c).all():
                return None
            lo, hi = int(c.min()), int(c.max())
            dt = _int_type(lo, hi, unsigned_ok=False)
            if dt is None:
                continue
            ci = c.astype(np.int64)
            if not np.array_equal((ci / s).view(np.int64), bits):
                continue
            stored = torch.from_numpy(ci).to(device=t.device, dtype=dt)
            decoded = project([decode_expr(stored, s)], None)[0]
            if not bool((decoded.view(torch.int64) == t.view(torch.int64)).all()):
                continue
            set_value_range(stored, lo, hi)
            return CompactSpec(dt, s), stored
    return None


def compact_column(col: EncodedTensor) -> EncodedTensor:
    """``col`` in compact storage when a lossless narrow form exists."""
    plan = plan_column(col)
    if plan is None:
        return col
    spec, stored = plan
    return from_stored(stored, spec, col)


def compact_table(table: Table) -> Table:
    """Ingestion-time compaction of every column of a table (values, logical
    types, encodings and query results unchanged)."""
    cols = [compact_column(c) for c in table.columns]
    return table_from_columns(list(table.schema.names), cols, device=table.device)


def stored_bytes(col: EncodedTensor) -> int:
    """Bytes per row the column occupies in storage."""
    v = col.values
    if v._t is None and isinstance(v._lazy, LazyValue):
        src = compact_source(v._lazy.expr)
        if src is not None:
            return src[0].element_size()
        if v._lazy.expr.op == "col":
            return v._lazy.expr.col.element_size()
    return v.data.element_size()


def specs_of(table: Table) -> list[Optional[CompactSpec]]:
    """Storage spec per column (None: stored at full width)."""
    out = []
    for c in table.columns:
        v = c.values
        src = compact_source(v._lazy.expr) if v._t is None and isinstance(v._lazy, LazyValue) else None
        out.append(CompactSpec(src[0].dtype, src[1]) if src is not None else None)
    return out


def stored_tensors(table: Table) -> list[torch.Tensor]:
    """The tensors a table's columns are stored in (narrow for compact columns)."""
    out = []
    for c in table.columns:
        v = c.values
        src = compact_source(v._lazy.expr) if v._t is None and isinstance(v._lazy, LazyValue) else None
        out.append(src[0] if src is not None else v.data)
    return out


def table_from_stored(like: Table, stored: Sequence[torch.Tensor]) -> Table:
    """A table with ``like``'s schema, encodings and storage specs over new
    stored tensors (one per column) -- e.g. the device copies of a compact
    table kept in pinned host memory."""
    cols = []
    for c, spec, t in zip(like.columns, specs_of(like), stored):
        if spec is None:
            with trusted():
                cols.append(EncodedTensor(Tensor(t), c.encoding))
        else:
            cols.append(from_stored(t, spec, c))
    return table_from_columns(list(like.schema.names), cols, device=like.device)

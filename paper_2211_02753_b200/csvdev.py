"""Device CSV ingestion (register_csv onto the device).

``read_csv_device(data, schema, ...)`` tokenises and converts a CSV file's
UTF-8 bytes on the GPU (``csrc/csv.cu``): record / field boundaries with a
speculative quote-parity scan, int64 and float64 cells parsed per row
(floats exact on the device on Clinger's fast path, the rest converted by
Python's ``float`` cell by cell), string cells unescaped into one byte
buffer and dictionary-encoded on the device (``strings.cu``).  It returns
None whenever the file needs the host reader's semantics -- anything the
device tokenizer does not model (stray quotes, empty lines, malformed
UTF-8), or any error the reference raises -- and the caller then runs the
host reader (``storage.read_csv``), which reproduces the reference's
(tq/storage.py:206-249) result or ``StorageError`` exactly.  Results equal
the host reader's bit for bit (tests/test_gpu_csv.py).
"""

from __future__ import annotations

import csv
from typing import Optional

import numpy as np

# below this many bytes the host reader is faster than the launches
DEVICE_CSV_MIN_BYTES = 1 << 16
INT32_MAX = 0x7FFFFFFF

# "device" / "host": which path the last read_csv / register_csv took (tests)
LAST_PATH = None


def read_csv_device(data: bytes, schema, device, source: str):
    """Table of ``data`` parsed on the device, or None (use the host reader)."""
    import torch

    from . import _native as nat
    from .encodings import dict_encode_device_bytes, plain
    from .hostread import read_ints
    from .storage import Table
    from .tensor import Tensor

    if len(data) < DEVICE_CSV_MIN_BYTES or not torch.cuda.is_available():
        return None
    kinds = [ctype.kind for _, ctype in schema.columns]
    if not kinds or any(k not in ("int", "float", "string") for k in kinds):
        return None
    if data[-1:] not in (b"\n", b"\r"):
        data = data + b"\n"
    dev = torch.device("cuda", torch.cuda.current_device())
    n = len(data)
    db = torch.from_numpy(np.frombuffer(data, dtype=np.uint8).copy()).to(dev)
    ws = nat.workspace(nat.load().tdp_csv_workspace(n), dev)
    counts = torch.empty(3, dtype=torch.int64, device=dev)
    nat.call("tdp_csv_index", nat.ptr(db), n, nat.ptr(counts), nat.ptr(ws), ws.numel(),
             nat.stream())
    nfields, nrec, nquotes = read_ints(counts)
    ncols = len(kinds)
    if nquotes % 2 or nrec < 1:
        return None
    fend = torch.empty(max(nfields, 1), dtype=torch.int64, device=dev)
    rend = torch.empty(max(nrec, 1), dtype=torch.int64, device=dev)
    flags = torch.empty(2, dtype=torch.int32, device=dev)
    nat.call("tdp_csv_fields", nat.ptr(db), n, ncols, nrec, nat.ptr(fend), nat.ptr(rend),
             nat.ptr(flags), nat.ptr(ws), ws.numel(), nat.stream())
    odd, bad_record = read_ints(flags)
    if odd or bad_record != INT32_MAX:
        return None
    # header: record 0, parsed by the csv module itself
    hdr_end = int(fend[ncols - 1].item())
    header = next(csv.reader([data[:hdr_end].decode("utf-8")]))
    if [h.strip() for h in header] != schema.names:
        return None
    nrows = nrec - 1
    if nrows == 0:
        return None  # header only: nothing to do on the device
    columns = []
    for j, (name, ctype) in enumerate(schema.columns):
        if ctype.kind == "string":
            col = _string_column(db, fend, ncols, j, nrows, dict_encode_device_bytes)
        else:
            col = _numeric_column(data, db, fend, ncols, j, nrows, ctype.kind)
        if col is None:
            return None
        columns.append(col if ctype.kind == "string" else plain(Tensor(col)))
    return Table(schema, tuple(columns), nrows, device)


def _numeric_column(data: bytes, db, fend, ncols: int, j: int, nrows: int, kind: str):
    import torch

    from . import _native as nat

    dev = db.device
    out = torch.empty(max(nrows, 1), dtype=torch.int64 if kind == "int" else torch.float64,
                      device=dev)
    status = torch.zeros(max(nrows, 1), dtype=torch.uint8, device=dev)
    nat.call("tdp_csv_parse_column", nat.ptr(db), nat.ptr(fend), ncols, j, nrows,
             0 if kind == "int" else 1, nat.ptr(out), nat.ptr(status), nat.stream())
    out = out[:nrows]
    rows = torch.nonzero(status[:nrows]).flatten()
    if rows.numel() == 0:
        return out
    st = status[rows].cpu().numpy()
    if (st == 2).any():
        return None  # an invalid cell: the host reader raises the reference's error
    # cells the device does not convert exactly: Python's int() / float()
    cell = (rows + 1) * ncols + j
    ends = fend[cell].cpu().numpy()
    prev = fend[cell - 1].cpu().numpy()
    conv = int if kind == "int" else float
    vals = []
    for p, e in zip(prev.tolist(), ends.tolist()):
        s = p + 1 + (1 if data[p:p + 2] == b"\r\n" else 0)
        text = data[s:e]
        if text[:1] == b'"':
            text = text[1:-1].replace(b'""', b'"')
        try:
            v = conv(text.decode("utf-8").strip())
        except ValueError:
            return None
        if kind == "int" and not -(1 << 63) <= v < (1 << 63):
            return None  # np.asarray raises OverflowError on the host path
        vals.append(v)
    out[rows] = torch.tensor(vals, dtype=out.dtype).to(dev)
    return out


def _string_column(db, fend, ncols: int, j: int, nrows: int, encode) -> Optional[object]:
    import torch

    from . import _native as nat
    from .hostread import read_ints

    dev = db.device
    offs = torch.empty(nrows + 1, dtype=torch.int64, device=dev)
    ws = nat.workspace(nat.load().tdp_csv_string_workspace(nrows), dev)
    nat.call("tdp_csv_string_column", nat.ptr(db), nat.ptr(fend), ncols, j, nrows, nat.ptr(offs),
             None, nat.ptr(ws), ws.numel(), nat.stream())
    total = read_ints(offs[nrows:])[0]
    sb = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
    nat.call("tdp_csv_string_column", nat.ptr(db), nat.ptr(fend), ncols, j, nrows, nat.ptr(offs),
             nat.ptr(sb), nat.ptr(ws), ws.numel(), nat.stream())
    return encode(sb, offs, nrows)

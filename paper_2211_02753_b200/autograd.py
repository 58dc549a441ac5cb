"""torch.autograd bindings of the differentiable B200 kernels.

Each Function's forward and backward call libtdp_kernels; PyTorch's autograd
engine only sequences them (it is the "tape" of this build).

* :func:`softmax_rows`   -- row softmax and its VJP (tq/tensor.py:515-527)
* :func:`gather_rows`    -- row gather and its scatter-add VJP (tq/tensor.py:597-614)
* :func:`soft_groupby_grid` -- soft grouped count / weighted sum over PE keys and
  its VJP (tq/kernels.py:190-229 and the reduce_sum/mul/reshape VJP chain).
* :func:`soft_linear_count` -- the soft count whose dense key is
  pe_encode(Linear(X)), fused into one pass over X forward and one backward.
"""

from __future__ import annotations

from ctypes import c_void_p
from typing import Optional, Sequence

import torch

from . import _native as nat


def _dt(t: torch.Tensor) -> int:
    return nat.TORCH_TO_TDP[t.dtype]


class _SoftmaxRows(torch.autograd.Function):
    @staticmethod
    def forward(ctx, logits: torch.Tensor) -> torch.Tensor:
        x = logits.contiguous()
        nat.require_cuda(x)
        n, k = x.shape
        out = torch.empty_like(x)
        nat.call("tdp_softmax_fwd", nat.ptr(x), _dt(x), n, k, nat.ptr(out), nat.stream())
        ctx.save_for_backward(out)
        return out

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        (p,) = ctx.saved_tensors
        g = g.contiguous().to(p.dtype)
        n, k = p.shape
        dz = torch.empty_like(p)
        nat.call("tdp_softmax_bwd", nat.ptr(p), nat.ptr(g), _dt(p), n, k, nat.ptr(dz), nat.stream())
        return dz


def softmax_rows(logits: torch.Tensor) -> torch.Tensor:
    return _SoftmaxRows.apply(logits)


def gather_rows_raw(x: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    """Row gather without autograd (B200 kernel)."""
    x = x.contiguous()
    nat.require_cuda(x, idx)
    m = idx.numel()
    out = torch.empty((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    if m:
        cols = nat.columns([x])
        dst = (c_void_p * 1)(out.data_ptr())
        nat.call("tdp_gather_rows", cols, 1, nat.ptr(idx), m, dst, nat.stream())
    return out


def gather_many(xs: Sequence[torch.Tensor], idx: torch.Tensor) -> list[torch.Tensor]:
    """Gather several columns with one index vector in a single launch."""
    nat.require_cuda(idx, *xs)
    m = idx.numel()
    outs = [torch.empty((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device) for x in xs]
    if m and xs:
        xs = [x.contiguous() for x in xs]
        cols = nat.columns(xs)
        dst = (c_void_p * len(xs))(*[o.data_ptr() for o in outs])
        nat.call("tdp_gather_rows", cols, len(xs), nat.ptr(idx), m, dst, nat.stream())
    return outs


class _GatherRows(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
        ctx.save_for_backward(idx)
        ctx.src_shape = tuple(x.shape)
        return gather_rows_raw(x, idx)

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        (idx,) = ctx.saved_tensors
        g = g.contiguous()
        out = torch.zeros(ctx.src_shape, dtype=g.dtype, device=g.device)
        m = idx.numel()
        width = 1
        for s in ctx.src_shape[1:]:
            width *= s
        if m:
            nat.call("tdp_scatter_add_rows", nat.ptr(g), _dt(g), width, nat.ptr(idx), m,
                     nat.ptr(out), nat.stream())
        return out, None


def gather_rows(x: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    if x.is_floating_point() and x.requires_grad:
        return _GatherRows.apply(x, idx)
    return gather_rows_raw(x, idx)


class _ColumnSum(torch.autograd.Function):
    """SUM of a 1-d float column on the fused scan kernel (float64
    accumulation, fixed reduction order); VJP: the upstream gradient
    broadcast to every row (tq/tensor.py:474)."""

    @staticmethod
    def forward(ctx, x: torch.Tensor) -> torch.Tensor:
        from .kernels import _scan_single

        ctx.n = x.shape[0]
        _, raw = _scan_single(x.detach())
        return raw.view(torch.float64).to(x.dtype).reshape(())

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        return g.reshape(1).expand(ctx.n).contiguous()


def column_sum(x: torch.Tensor) -> torch.Tensor:
    """Differentiable sum of a 1-d float CUDA column (0-d result, input dtype)."""
    return _ColumnSum.apply(x)


# ---------------------------------------------------------------------------
# skinny linear layer (matmul with few output columns)
# ---------------------------------------------------------------------------

LINEAR_MAX_K = 8
LINEAR_MAX_D = 256
LINEAR_MIN_ROWS = 1 << 14


def linear_eligible(a: torch.Tensor, b: torch.Tensor) -> bool:
    """Tall-skinny products the streaming kernels handle (else cuBLAS)."""
    return (a.is_cuda and b.is_cuda and a.dim() == 2 and b.dim() == 2
            and a.dtype == b.dtype and a.dtype in (torch.float32, torch.float64)
            and 1 <= b.shape[1] <= LINEAR_MAX_K and 1 <= a.shape[1] <= LINEAR_MAX_D
            and a.shape[0] >= LINEAR_MIN_ROWS)


class _SkinnyLinear(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x: torch.Tensor, w: torch.Tensor, b: Optional[torch.Tensor]) -> torch.Tensor:
        x = x.contiguous()
        w = w.contiguous()
        b = None if b is None else b.contiguous()
        n, d = x.shape
        k = w.shape[1]
        y = torch.empty((n, k), dtype=x.dtype, device=x.device)
        nat.call("tdp_linear_fwd", nat.ptr(x), _dt(x), n, d, k, nat.ptr(w), nat.ptr(b),
                 nat.ptr(y), nat.stream())
        ctx.save_for_backward(x, w)
        ctx.has_bias = b is not None
        return y

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        x, w = ctx.saved_tensors
        g = g.contiguous().to(x.dtype)
        n, d = x.shape
        k = w.shape[1]
        dx = dw = db = None
        if ctx.needs_input_grad[0]:
            dx = torch.matmul(g, w.t())
        want_b = ctx.has_bias and ctx.needs_input_grad[2]
        if ctx.needs_input_grad[1] or want_b:
            dw = torch.empty_like(w)
            db = torch.empty(k, dtype=x.dtype, device=x.device) if want_b else None
            ws = nat.workspace(nat.load().tdp_linear_wgrad_workspace(n, d, k), x.device)
            nat.call("tdp_linear_wgrad", nat.ptr(x), nat.ptr(g), _dt(x), n, d, k, nat.ptr(dw),
                     nat.ptr(db), nat.ptr(ws), ws.numel(), nat.stream())
            if not ctx.needs_input_grad[1]:
                dw = None
        return dx, dw, db


def skinny_linear(x: torch.Tensor, w: torch.Tensor, b: Optional[torch.Tensor] = None) -> torch.Tensor:
    return _SkinnyLinear.apply(x, w, b)


# ---------------------------------------------------------------------------
# soft group-by
# ---------------------------------------------------------------------------

class SoftKeySpec:
    """Static description of the key list: ('dense', k) or ('onehot', k) per key."""

    def __init__(self, kinds: Sequence[tuple[str, int]]):
        self.kinds = tuple(kinds)

    @property
    def cells(self) -> int:
        c = 1
        for _, k in self.kinds:
            c *= k
        return c


def _soft_keys(spec: SoftKeySpec, tensors: Sequence[torch.Tensor]):
    arr = (nat.SoftKey * len(tensors))()
    for j, ((kind, k), t) in enumerate(zip(spec.kinds, tensors)):
        if kind == "dense":
            arr[j] = nat.SoftKey(c_void_p(t.data_ptr()), nat.SOFT_DENSE, _dt(t), k)
        else:
            arr[j] = nat.SoftKey(c_void_p(t.data_ptr()), nat.SOFT_ONEHOT, nat.I64, k)
    return arr


class _SoftGroupBy(torch.autograd.Function):
    @staticmethod
    def forward(ctx, spec: SoftKeySpec, n: int, out_dtype: torch.dtype, values: Optional[torch.Tensor],
                *keys: torch.Tensor):
        keys = tuple(k.contiguous() for k in keys)
        nat.require_cuda(*keys)
        dev = keys[0].device
        grid = torch.empty(spec.cells, dtype=torch.float64, device=dev)
        vals = None if values is None else values.contiguous()
        nat.call("tdp_soft_groupby_fwd", _soft_keys(spec, keys), len(keys), n, nat.ptr(vals),
                 nat.I64 if vals is None else _dt(vals), nat.ptr(grid), nat.stream())
        ctx.spec = spec
        ctx.n = n
        ctx.has_values = vals is not None
        ctx.save_for_backward(*(keys + ((vals,) if vals is not None else ())))
        return grid.to(out_dtype)

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        saved = ctx.saved_tensors
        spec = ctx.spec
        nk = len(spec.kinds)
        keys = saved[:nk]
        vals = saved[nk] if ctx.has_values else None
        G = g.detach().to(torch.float64).contiguous()
        grads: list[Optional[torch.Tensor]] = [None] * nk
        ptrs = (c_void_p * nk)()
        for j, ((kind, _), t) in enumerate(zip(spec.kinds, keys)):
            if kind == "dense" and ctx.needs_input_grad[4 + j]:
                grads[j] = torch.empty_like(t)
                ptrs[j] = grads[j].data_ptr()
        dvals = None
        if vals is not None and ctx.needs_input_grad[3]:
            dvals = torch.empty_like(vals)
        if any(x is not None for x in grads) or dvals is not None:
            nat.call("tdp_soft_groupby_bwd", _soft_keys(spec, keys), nk, ctx.n, nat.ptr(vals),
                     nat.I64 if vals is None else _dt(vals), nat.ptr(G), ptrs, nat.ptr(dvals),
                     nat.stream())
        return (None, None, None, dvals, *grads)


def soft_groupby_grid(spec: SoftKeySpec, keys: Sequence[torch.Tensor], n: int,
                      out_dtype: torch.dtype, values: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Dense grid (flattened, row-major over keys) of sum_i w_i prod_j P_j[i, c_j]."""
    return _SoftGroupBy.apply(spec, n, out_dtype, values, *keys)


# ---------------------------------------------------------------------------
# fused soft count over a linear classifier head (LLP)
# ---------------------------------------------------------------------------

def soft_linear_supported(x: torch.Tensor, w: torch.Tensor, cells: int) -> bool:
    """Shapes the fused kernels cover (tdp_soft_linear_supported)."""
    if not (x.is_cuda and x.dim() == 2 and w.dim() == 2 and x.dtype == w.dtype
            and x.dtype in (torch.float32, torch.float64) and x.is_contiguous()):
        return False
    return bool(nat.load().tdp_soft_linear_supported(_dt(x), x.shape[0], x.shape[1], w.shape[1],
                                                     int(cells), nat.ptr(x)))


def linear_keys(spec: SoftKeySpec, dense_pos: int, codes: Sequence[torch.Tensor]):
    arr = (nat.SoftKey * len(spec.kinds))()
    it = iter(codes)
    for j, (kind, k) in enumerate(spec.kinds):
        if j == dense_pos:
            arr[j] = nat.SoftKey(None, nat.SOFT_DENSE, nat.F32, k)
        else:
            arr[j] = nat.SoftKey(c_void_p(next(it).data_ptr()), nat.SOFT_ONEHOT, nat.I64, k)
    return arr


def bag_index(codes: torch.Tensor, bags: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Rows of a one-hot key column in bag order: (int32 stable permutation,
    int64 offsets [bags + 1]).  Built once per code column with the radix sort
    and cached on it (valid while its in-place version is unchanged), like an
    index on the column."""
    meta = getattr(codes, "_tdp_bag_index", None)
    if meta is not None and meta[0] == codes._version and meta[1] == bags:
        return meta[2], meta[3]
    from .encodings import plain
    from .kernels import _groupby_codes, stable_order
    from .tensor import Tensor

    n = int(codes.numel())
    perm = stable_order(plain(Tensor(codes))).to(torch.int32)
    counts, _ = _groupby_codes(codes, bags, [], [], n, codes.device)
    offs = torch.zeros(bags + 1, dtype=torch.int64, device=codes.device)
    offs[1:] = torch.cumsum(counts, 0)
    codes._tdp_bag_index = (codes._version, bags, perm, offs)
    return perm, offs


def _onepass_layout(spec: SoftKeySpec, dense_pos: int, x: torch.Tensor, w: torch.Tensor,
                    codes) -> Optional[tuple[int, int, int]]:
    """(bags, bag stride, dense stride) when the one-pass LLP step applies:
    float32 X with 32 or 64 features, two classes, one one-hot key (SURVEY
    §8(f) 3, llp_onepass.cu); None otherwise (the two-pass kernels)."""
    import os

    if os.environ.get("TDP_LLP_ONEPASS", "1") == "0":
        return None
    if not (x.dtype == torch.float32 and x.shape[1] in (32, 64) and w.shape[1] == 2
            and len(codes) == 1 and len(spec.kinds) == 2 and x.shape[0] < (1 << 31)
            and x.data_ptr() % 16 == 0):
        return None
    strides, st = [0, 0], 1
    for j in (1, 0):
        strides[j] = st
        st *= spec.kinds[j][1]
    bag_pos = 1 - dense_pos
    return spec.kinds[bag_pos][1], strides[bag_pos], strides[dense_pos]


class _SoftLinearCount(torch.autograd.Function):
    @staticmethod
    def forward(ctx, spec: SoftKeySpec, dense_pos: int, out_dtype: torch.dtype, x: torch.Tensor,
                w: torch.Tensor, b: Optional[torch.Tensor], *codes: torch.Tensor):
        x = x.contiguous()
        w = w.detach().contiguous()
        b = None if b is None else b.detach().contiguous()
        n, d = x.shape
        k = w.shape[1]
        grid = torch.empty(spec.cells, dtype=torch.float64, device=x.device)
        ctx.spec, ctx.dense_pos, ctx.has_bias = spec, dense_pos, b is not None
        onepass = _onepass_layout(spec, dense_pos, x, w, codes)
        if onepass is not None:
            # one pass over X: the grid and the per-bag statistics of the
            # backward (llp_onepass.cu); the backward never reads X
            bags, bag_stride, dense_stride = onepass
            perm, offs = bag_index(codes[0].contiguous(), bags)
            stats = torch.empty((bags, d + 1), dtype=torch.float64, device=x.device)
            ws = nat.workspace(nat.load().tdp_llp_onepass_workspace(bags, d), x.device)
            nat.call("tdp_llp_onepass_fwd", nat.ptr(x), n, d, nat.ptr(w), nat.ptr(b), nat.ptr(perm),
                     nat.ptr(offs), bags, bag_stride, dense_stride, nat.ptr(grid), nat.ptr(stats),
                     nat.ptr(ws), ws.numel(), nat.stream())
            ctx.onepass = (bags, bag_stride, dense_stride, d)
            ctx.save_for_backward(stats, w, *(() if b is None else (b,)))
            return grid.to(out_dtype)
        ctx.onepass = None
        keys = linear_keys(spec, dense_pos, codes)
        nat.call("tdp_soft_linear_count_fwd", nat.ptr(x), _dt(x), n, d, k, nat.ptr(w), nat.ptr(b),
                 keys, len(spec.kinds), dense_pos, nat.ptr(grid), nat.stream())
        ctx.save_for_backward(x, w, *(() if b is None else (b,)), *codes)
        return grid.to(out_dtype)

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        if ctx.onepass is not None:
            saved = ctx.saved_tensors
            stats, w = saved[0], saved[1]
            b = saved[2] if ctx.has_bias else None
            bags, bag_stride, dense_stride, d = ctx.onepass
            G = g.detach().to(torch.float64).contiguous()
            dw = torch.empty_like(w)
            db = torch.empty_like(b) if b is not None else None
            nat.call("tdp_llp_onepass_bwd", nat.ptr(stats), bags, d, nat.ptr(G), bag_stride,
                     dense_stride, nat.ptr(dw), nat.ptr(db), nat.stream())
            return (None, None, None, None, dw if ctx.needs_input_grad[4] else None,
                    db if ctx.has_bias and ctx.needs_input_grad[5] else None,
                    *([None] * (len(ctx.needs_input_grad) - 6)))
        saved = ctx.saved_tensors
        x, w = saved[0], saved[1]
        b = saved[2] if ctx.has_bias else None
        codes = saved[3 if ctx.has_bias else 2:]
        n, d = x.shape
        k = w.shape[1]
        G = g.detach().to(torch.float64).contiguous()
        dw = torch.empty_like(w)
        db = torch.empty_like(b) if b is not None else None
        ws = nat.workspace(nat.load().tdp_soft_linear_count_bwd_workspace(n, d, k), x.device)
        keys = linear_keys(ctx.spec, ctx.dense_pos, codes)
        nat.call("tdp_soft_linear_count_bwd", nat.ptr(x), _dt(x), n, d, k, nat.ptr(w), nat.ptr(b),
                 keys, len(ctx.spec.kinds), ctx.dense_pos, nat.ptr(G), nat.ptr(dw), nat.ptr(db),
                 nat.ptr(ws), ws.numel(), nat.stream())
        return (None, None, None, None, dw if ctx.needs_input_grad[4] else None,
                db if ctx.has_bias and ctx.needs_input_grad[5] else None,
                *([None] * len(codes)))


# ---------------------------------------------------------------------------
# wide heads: softmax(X W + b) with n x k logits too large to form at once
# (SURVEY §8(d) 4': Linear(64, 1000) over 1e8 rows = 400 GB of logits)
# ---------------------------------------------------------------------------
WIDE_HEAD_BYTES = 8 << 30   # defer a Linear whose logits would exceed this
CHUNK_BYTES = 1 << 30       # logits formed per chunk of rows


def wide_head(x: torch.Tensor, w: torch.Tensor) -> bool:
    """A constant-input linear head whose logits exceed WIDE_HEAD_BYTES."""
    return (x.is_cuda and w.is_cuda and x.dim() == 2 and w.dim() == 2 and not x.requires_grad
            and x.dtype == w.dtype and x.dtype in (torch.float32, torch.float64)
            and x.shape[0] * w.shape[1] * x.element_size() > WIDE_HEAD_BYTES)


def _chunk_keys(spec: SoftKeySpec, dense_pos: int, codes, lo: int, hi: int, p: torch.Tensor):
    it = iter(codes)
    keys = []
    for j, (kind, _) in enumerate(spec.kinds):
        keys.append(p if j == dense_pos else next(it)[lo:hi])
    return keys


class _ChunkedSoftLinearCount(torch.autograd.Function):
    """Soft COUNT over one key P = softmax(X W + b) (x one-hot keys) whose
    logits are never formed in full: rows in chunks of CHUNK_BYTES of logits,
    each chunk's logits by cuBLAS (bias as a column of ones; no TF32),
    softmaxed and counted (tdp_softmax_fwd; column sums for a single key,
    tdp_soft_groupby_fwd with one-hot keys)
    into the grid; the backward recomputes each chunk's P and forms
    dZ = softmax VJP of the gathered grid gradient (tdp_soft_groupby_bwd,
    tdp_softmax_bwd), dW += X_c^T dZ, db += sum dZ (tq/tensor.py:474,
    :364-365, :515-527, :437-447)."""

    @staticmethod
    def forward(ctx, spec: SoftKeySpec, dense_pos: int, out_dtype: torch.dtype, x: torch.Tensor,
                w: torch.Tensor, b: Optional[torch.Tensor], *codes: torch.Tensor):
        x, wd = x.contiguous(), w.detach().contiguous()
        bd = None if b is None else b.detach().contiguous()
        n, k = x.shape[0], wd.shape[1]
        rows = max(1, CHUNK_BYTES // (k * x.element_size()))
        grid = torch.zeros(spec.cells, dtype=torch.float64, device=x.device)
        part = torch.empty_like(grid)
        for lo in range(0, n, rows):
            hi = min(n, lo + rows)
            p = _chunk_softmax(x[lo:hi], wd, bd)
            if len(spec.kinds) == 1:  # one key: the grid is P's column sums
                grid += _colsum64(p)
                continue
            keys = _chunk_keys(spec, dense_pos, codes, lo, hi, p)
            nat.call("tdp_soft_groupby_fwd", _soft_keys(spec, keys), len(keys), hi - lo, None,
                     nat.I64, nat.ptr(part), nat.stream())
            grid += part
        ctx.spec, ctx.dense_pos, ctx.rows, ctx.has_bias = spec, dense_pos, rows, b is not None
        ctx.save_for_backward(x, w, *(() if b is None else (b,)), *codes)
        return grid.to(out_dtype)

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        saved = ctx.saved_tensors
        x, w = saved[0], saved[1]
        b = saved[2] if ctx.has_bias else None
        codes = saved[3 if ctx.has_bias else 2:]
        wd = w.detach().contiguous()
        bd = None if b is None else b.detach().contiguous()
        spec, pos = ctx.spec, ctx.dense_pos
        G = g.detach().to(torch.float64).contiguous()
        n, k = x.shape[0], wd.shape[1]
        dw = torch.zeros(wd.shape, dtype=torch.float64, device=x.device)
        db = torch.zeros(k, dtype=torch.float64, device=x.device)
        nk = len(spec.kinds)
        for lo in range(0, n, ctx.rows):
            hi = min(n, lo + ctx.rows)
            xc = x[lo:hi]
            p = _chunk_softmax(xc, wd, bd)
            keys = _chunk_keys(spec, pos, codes, lo, hi, p)
            dp = torch.empty_like(p)
            ptrs = (c_void_p * nk)()
            ptrs[pos] = dp.data_ptr()
            nat.call("tdp_soft_groupby_bwd", _soft_keys(spec, keys), nk, hi - lo, None, nat.I64,
                     nat.ptr(G), ptrs, None, nat.stream())
            dz = torch.empty_like(p)
            nat.call("tdp_softmax_bwd", nat.ptr(p), nat.ptr(dp), _dt(p), hi - lo, k, nat.ptr(dz),
                     nat.stream())
            dw += (xc.t() @ dz).to(torch.float64)
            db += _colsum64(dz)
        gw = dw.to(w.dtype) if ctx.needs_input_grad[4] else None
        gb = db.to(b.dtype) if b is not None and ctx.needs_input_grad[5] else None
        return (None, None, None, None, gw, gb, *([None] * len(codes)))


def _colsum64(t: torch.Tensor, group: int = 256) -> torch.Tensor:
    """Column sums of a [rows, k] chunk in float64: groups of ``group`` rows
    summed in the chunk's dtype (no float64 copy of the chunk), the group sums
    in float64."""
    rows = t.shape[0] - t.shape[0] % group
    out = torch.zeros(t.shape[1], dtype=torch.float64, device=t.device)
    if rows:
        out += t[:rows].view(-1, group, t.shape[1]).sum(1).sum(0, dtype=torch.float64)
    if rows < t.shape[0]:
        out += t[rows:].sum(0, dtype=torch.float64)
    return out


def _chunk_softmax(xc: torch.Tensor, w: torch.Tensor, b: Optional[torch.Tensor]) -> torch.Tensor:
    # the bias rides in the GEMM as a column of ones (no pass over the
    # chunk's logits to add it: x.w + b rounded once)
    if b is not None:
        xc = torch.cat([xc, torch.ones((xc.shape[0], 1), dtype=xc.dtype, device=xc.device)], 1)
        w = torch.cat([w, b.reshape(1, -1)], 0)
    z = torch.matmul(xc, w)
    p = torch.empty_like(z)
    nat.call("tdp_softmax_fwd", nat.ptr(z), _dt(z), z.shape[0], z.shape[1], nat.ptr(p),
             nat.stream())
    return p


def chunked_soft_linear_count(spec: SoftKeySpec, dense_pos: int, codes: Sequence[torch.Tensor],
                              x: torch.Tensor, w: torch.Tensor, b: Optional[torch.Tensor],
                              out_dtype: torch.dtype) -> torch.Tensor:
    return _ChunkedSoftLinearCount.apply(spec, dense_pos, out_dtype, x, w, b, *codes)


def soft_linear_count(spec: SoftKeySpec, dense_pos: int, codes: Sequence[torch.Tensor],
                      x: torch.Tensor, w: torch.Tensor, b: Optional[torch.Tensor],
                      out_dtype: torch.dtype) -> torch.Tensor:
    """Flattened count grid of softmax(x w + b) crossed with one-hot keys."""
    return _SoftLinearCount.apply(spec, dense_pos, out_dtype, x, w, b, *codes)


# ---------------------------------------------------------------------------
# differentiable ORDER BY: NeuralSort relaxation
# ---------------------------------------------------------------------------

class _SoftSort(torch.autograd.Function):
    """P [k, n]: row r the relaxed one-hot of the rank-r (descending) row of
    scores s (float64), temperature tau (csrc/softsort.cu)."""

    @staticmethod
    def forward(ctx, s: torch.Tensor, k: int, tau: float) -> torch.Tensor:
        s = s.detach().to(torch.float64).contiguous()
        n = s.numel()
        P = torch.empty((k, n), dtype=torch.float64, device=s.device)
        ws = torch.empty(max(n, 1), dtype=torch.float64, device=s.device)
        nat.call("tdp_softsort_fwd", nat.ptr(s), n, k, float(tau), nat.ptr(P), nat.ptr(ws),
                 nat.stream())
        ctx.tau, ctx.k = tau, k
        ctx.save_for_backward(s, P)
        return P

    @staticmethod
    def backward(ctx, dP: torch.Tensor):
        s, P = ctx.saved_tensors
        n = s.numel()
        g = dP.detach().to(torch.float64).contiguous().clone()
        ds = torch.empty(n, dtype=torch.float64, device=s.device)
        ws = torch.empty(2 * max(n, 1), dtype=torch.float64, device=s.device)
        nat.call("tdp_softsort_bwd", nat.ptr(s), n, ctx.k, float(ctx.tau), nat.ptr(P), nat.ptr(g),
                 nat.ptr(ds), nat.ptr(ws), nat.stream())
        return ds, None, None


def soft_sort_matrix(s: torch.Tensor, k: int, tau: float) -> torch.Tensor:
    """Relaxed top-k permutation rows of the scores (descending)."""
    return _SoftSort.apply(s, k, tau)

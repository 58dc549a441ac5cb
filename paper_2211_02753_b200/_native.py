"""ctypes binding of libtdp_kernels.so (the C ABI in include/tdp_kernels.h).

This module is the only place the host layer touches the native library.  It
translates device ``torch.Tensor`` arguments into the plain-pointer
descriptors of the C ABI, passes the current CUDA stream, and turns negative
status codes into :class:`NativeError` carrying ``tdp_last_error()``.

There is no CPU implementation behind any of these calls: a tensor that is
not on a CUDA device, or a missing library, raises immediately.
"""

from __future__ import annotations

import ctypes
import threading
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t, c_uint64, c_void_p
from pathlib import Path
from typing import Optional, Sequence

import torch

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libtdp_kernels.so"

# status codes (include/tdp_kernels.h)
TDP_OK, TDP_EINVAL, TDP_ECUDA, TDP_ENOMEM, TDP_ENOTSUP, TDP_EJIT = 0, -1, -2, -3, -4, -5

# dtypes
I64, F64, F32, BOOL, I32 = 0, 1, 2, 3, 4
I8, I16, U8 = 5, 6, 7  # compact storage widths (compact.py)
TORCH_TO_TDP = {torch.int64: I64, torch.float64: F64, torch.float32: F32, torch.bool: BOOL,
                torch.int32: I32, torch.int8: I8, torch.int16: I16, torch.uint8: U8}
NAME_TO_TDP = {"int64": I64, "float64": F64, "float32": F32, "bool": BOOL}

# comparison ops / kinds
CMP_OPS = {"=": 0, "<>": 1, "<": 2, ">": 3, "<=": 4, ">=": 5}
CMP_I64, CMP_F64, CMP_F32, CMP_NONE, CMP_ALL, CMP_DEC, CMP_BITMAP = 0, 1, 2, 3, 4, 5, 6

# expression opcodes
OP_LOAD, OP_CONST, OP_CAST, OP_ADD, OP_SUB, OP_MUL, OP_DIV = 0, 1, 2, 3, 4, 5, 6
OP_NEG, OP_SQUARE, OP_LOG, OP_EXP, OP_RELU, OP_DECIMAL = 7, 8, 9, 10, 11, 12

AGG_COUNT, AGG_SUM_F64, AGG_SUM_I64 = 0, 1, 2
AGG_AVG_BIT = 0x100  # group-by emit: write the float64 mean (TDP_AGG_AVG_BIT)
SOFT_DENSE, SOFT_ONEHOT = 0, 1


class NativeError(RuntimeError):
    """A libtdp_kernels call failed (bad descriptor, CUDA or NVRTC error)."""


class Column(ctypes.Structure):
    _fields_ = [("data", c_void_p), ("dtype", c_int32), ("reserved", c_int32),
                ("rows", c_int64), ("width", c_int64)]


class Predicate(ctypes.Structure):
    _fields_ = [("column", c_int32), ("op", c_int32), ("cmp", c_int32), ("reserved", c_int32),
                ("lit_i", c_int64), ("lit_f", c_double)]


class Instr(ctypes.Structure):
    _fields_ = [("op", c_int32), ("dtype", c_int32), ("a", c_int32), ("b", c_int32),
                ("imm_i", c_int64), ("imm_f", c_double)]


class Key(ctypes.Structure):
    _fields_ = [("value", c_int32), ("reserved", c_int32), ("lo", c_int64), ("span", c_int64)]


class Agg(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("value", c_int32)]


class SoftKey(ctypes.Structure):
    _fields_ = [("data", c_void_p), ("kind", c_int32), ("dtype", c_int32), ("k", c_int64)]


_SIGNATURES = {
    "tdp_last_error": (c_char_p, []),
    "tdp_version": (c_char_p, []),
    "tdp_device_sm_count": (c_int, []),
    "tdp_launch_count": (c_uint64, []),
    "tdp_count_graph_launches": (None, [c_uint64]),
    "tdp_stream_wait_event": (c_int, [c_void_p, c_void_p]),
    "tdp_replay_done": (c_int, [c_void_p, c_void_p, c_uint64]),
    "tdp_clear_error": (c_int, []),
    "tdp_expect_values": (c_int, [c_void_p, c_int32, c_int32, c_void_p, c_void_p]),
    "tdp_replay_log_begin": (c_int, [c_int32, c_void_p, c_int64]),
    "tdp_replay_log_size": (c_int64, []),
    "tdp_replay_log_end": (c_int, [c_void_p, c_int64]),
    "tdp_kernel_timer_enable": (c_int, [c_int32]),
    "tdp_kernel_timer_read": (c_int, [POINTER(c_double), POINTER(c_int64)]),
    "tdp_filter_mask": (c_int, [POINTER(Column), c_int32, POINTER(Predicate), c_int32, c_int64,
                                c_void_p, c_void_p]),
    "tdp_filter_workspace": (c_size_t, [c_int64]),
    "tdp_filter_select": (c_int, [POINTER(Column), c_int32, POINTER(Predicate), c_int32, c_int64,
                                  c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "tdp_gather_rows": (c_int, [POINTER(Column), c_int32, c_void_p, c_int64, POINTER(c_void_p),
                                c_void_p]),
    "tdp_gather_rows2": (c_int, [POINTER(Column), c_int32, c_int32, c_void_p, c_void_p, c_int64,
                                 POINTER(c_void_p), c_void_p]),
    "tdp_scatter_add_rows": (c_int, [c_void_p, c_int32, c_int64, c_void_p, c_int64, c_void_p,
                                     c_void_p]),
    "tdp_scan_aggregate_workspace": (c_size_t, [c_int64, c_int64, c_int32]),
    "tdp_scan_aggregate": (c_int, [POINTER(Column), c_int32, c_int64, POINTER(Predicate), c_int32,
                                   POINTER(Instr), c_int32, POINTER(Key), c_int32, POINTER(Agg),
                                   c_int32, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "tdp_scan_aggregate_grouped": (c_int, [POINTER(Column), c_int32, c_int64, POINTER(Predicate),
                                           c_int32, POINTER(Instr), c_int32, POINTER(Key), c_int32,
                                           POINTER(Agg), c_int32, c_void_p, c_void_p, c_void_p,
                                           c_size_t, c_uint64, c_void_p, c_void_p, c_void_p,
                                           c_void_p, c_void_p]),
    "tdp_scan_project": (c_int, [POINTER(Column), c_int32, c_int64, POINTER(Predicate), c_int32,
                                 POINTER(Instr), c_int32, POINTER(c_int32), c_int32,
                                 POINTER(c_void_p), c_void_p, c_void_p, c_size_t, c_void_p]),
    "tdp_pipeline_codegen": (c_int, [POINTER(Column), c_int32, c_int64, POINTER(Predicate),
                                     c_int32, POINTER(Instr), c_int32, POINTER(Key), c_int32,
                                     POINTER(Agg), c_int32, POINTER(c_int32), c_int32, c_int32,
                                     c_char_p, c_size_t]),
    "tdp_groupby_finalize": (c_int, [c_void_p, c_void_p, c_int64, POINTER(Key), c_int32,
                                     POINTER(Agg), c_int32, c_uint64, c_void_p, c_void_p,
                                     c_void_p, c_void_p, c_void_p]),
    "tdp_scan_minmax": (c_int, [POINTER(Column), c_int32, c_int64, POINTER(Predicate), c_int32,
                                POINTER(c_int32), c_int32, c_void_p, c_void_p]),
    "tdp_scan_minmax_runs": (c_int, [POINTER(Column), c_int32, c_int64, POINTER(Predicate),
                                     c_int32, POINTER(c_int32), c_int32, c_void_p, c_void_p,
                                     c_void_p]),
    "tdp_groupby_runs_workspace": (c_size_t, [c_int64]),
    "tdp_groupby_runs_prepare": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_size_t,
                                         c_void_p]),
    "tdp_groupby_runs_emit": (c_int, [c_void_p, c_int64, POINTER(Column), POINTER(c_int32),
                                      c_int32, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_size_t, c_void_p]),
    "tdp_sort_workspace": (c_size_t, [c_int64]),
    "tdp_topk_workspace": (c_size_t, [c_int64, c_int64]),
    "tdp_topk_order": (c_int, [POINTER(Column), c_int32, c_int64, c_int64, c_void_p, c_void_p,
                               c_size_t, c_void_p]),
    "tdp_sort_order": (c_int, [POINTER(Column), c_int32, c_int64, c_void_p, c_void_p, c_size_t,
                               c_void_p]),
    "tdp_unique_inverse": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_size_t, c_void_p]),
    "tdp_groupby_codes_workspace": (c_size_t, [c_int64, c_int32]),
    "tdp_groupby_codes": (c_int, [c_void_p, c_int64, c_int64, POINTER(Column), POINTER(c_int32),
                                  c_int32, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "tdp_groupby_hash_workspace": (c_size_t, [c_int64, c_int32]),
    "tdp_groupby_hash_prepare": (c_int, [c_void_p, c_int64, POINTER(Column), POINTER(c_int32),
                                         c_int32, c_void_p, c_void_p, c_size_t, c_void_p]),
    "tdp_groupby_hash_emit": (c_int, [c_int64, POINTER(c_int32), c_int32, c_int64, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "tdp_groupby_hash_prepare_ex": (c_int, [c_void_p, c_int64, POINTER(Column), POINTER(c_int32),
                                            c_int32, c_void_p, c_void_p, c_size_t, c_void_p]),
    "tdp_groupby_hash_rank_workspace": (c_size_t, [c_int64]),
    "tdp_groupby_hash_emit_ranked": (c_int, [c_int64, POINTER(c_int32), c_int32, c_int64, c_int64,
                                             c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                             c_size_t, c_void_p, c_size_t, c_void_p]),
    "tdp_join_workspace": (c_size_t, [c_int64, c_int64]),
    "tdp_join_prepare": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                                 c_size_t, c_void_p]),
    "tdp_join_prepare_filtered": (c_int, [c_void_p, c_int64, c_void_p, c_int64, POINTER(Column),
                                          c_int32, POINTER(Predicate), c_int32, c_void_p,
                                          c_void_p, c_size_t, c_void_p]),
    "tdp_join_prepare_ex": (c_int, [c_void_p, c_int64, POINTER(Column), c_int32,
                                    POINTER(Predicate), c_int32, c_void_p, c_int64,
                                    POINTER(Column), c_int32, POINTER(Predicate), c_int32, c_int32,
                                    c_void_p, c_void_p, c_size_t, c_void_p]),
    "tdp_join_emit": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_size_t,
                              c_void_p]),
    "tdp_string_hash": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "tdp_string_groups": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p,
                                  c_void_p, c_void_p]),
    "tdp_softsort_fwd": (c_int, [c_void_p, c_int64, c_int32, c_double, c_void_p, c_void_p,
                                 c_void_p]),
    "tdp_softsort_bwd": (c_int, [c_void_p, c_int64, c_int32, c_double, c_void_p, c_void_p,
                                 c_void_p, c_void_p, c_void_p]),
    "tdp_groupby_bitmap_workspace": (c_size_t, [c_int64, c_int64, c_int32]),
    "tdp_groupby_bitmap_prepare": (c_int, [c_void_p, c_int64, c_int64, c_int64, POINTER(Column),
                                           POINTER(c_int32), c_int32, c_void_p, c_void_p,
                                           c_size_t, c_void_p]),
    "tdp_groupby_bitmap_emit": (c_int, [c_int64, c_int64, c_int64, POINTER(c_int32), c_int32,
                                        c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_size_t, c_void_p]),
    "tdp_llp_onepass_workspace": (c_size_t, [c_int32, c_int32]),
    "tdp_llp_onepass_fwd": (c_int, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p,
                                    c_void_p, c_int32, c_int64, c_int64, c_void_p, c_void_p,
                                    c_void_p, c_size_t, c_void_p]),
    "tdp_llp_onepass_bwd": (c_int, [c_void_p, c_int32, c_int32, c_void_p, c_int64, c_int64,
                                    c_void_p, c_void_p, c_void_p]),
    "tdp_join_dense_workspace": (c_size_t, [c_int64, c_int64, c_int64]),
    "tdp_join_dense_prepare": (c_int, [c_void_p, c_int64, POINTER(Column), c_int32,
                                       POINTER(Predicate), c_int32, c_void_p, c_int64,
                                       POINTER(Column), c_int32, POINTER(Predicate), c_int32,
                                       c_int64, c_int64, c_int32, c_void_p, c_void_p, c_size_t,
                                       c_void_p]),
    "tdp_join_dense_bitmap": (c_int, [c_void_p, c_int64, POINTER(Column), c_int32,
                                      POINTER(Predicate), c_int32, c_int64, c_int64, c_void_p,
                                      c_void_p, c_void_p]),
    "tdp_join_dense_emit": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_int64, c_int32,
                                    c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "tdp_csv_workspace": (c_size_t, [c_int64]),
    "tdp_csv_string_workspace": (c_size_t, [c_int64]),
    "tdp_csv_index": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_size_t, c_void_p]),
    "tdp_csv_fields": (c_int, [c_void_p, c_int64, c_int32, c_int64, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_size_t, c_void_p]),
    "tdp_csv_parse_column": (c_int, [c_void_p, c_void_p, c_int32, c_int32, c_int64, c_int32,
                                     c_void_p, c_void_p, c_void_p]),
    "tdp_csv_string_column": (c_int, [c_void_p, c_void_p, c_int32, c_int32, c_int64, c_void_p,
                                      c_void_p, c_void_p, c_size_t, c_void_p]),
    "tdp_join_sorted_workspace": (c_size_t, [c_int64, c_int64]),
    "tdp_join_sorted_prepare": (c_int, [c_void_p, c_int64, c_void_p, c_int64, POINTER(Column),
                                        c_int32, POINTER(Predicate), c_int32, c_void_p, c_void_p,
                                        c_size_t, c_void_p]),
    "tdp_join_sorted_emit": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                     c_size_t, c_void_p]),
    "tdp_softmax_fwd": (c_int, [c_void_p, c_int32, c_int64, c_int64, c_void_p, c_void_p]),
    "tdp_softmax_bwd": (c_int, [c_void_p, c_void_p, c_int32, c_int64, c_int64, c_void_p,
                                c_void_p]),
    "tdp_pe_validate": (c_int, [c_void_p, c_int32, c_int64, c_int64, c_double, c_void_p,
                                c_void_p]),
    "tdp_pe_argmax": (c_int, [c_void_p, c_int32, c_int64, c_int64, c_void_p, c_void_p]),
    "tdp_codes_check": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "tdp_soft_groupby_fwd": (c_int, [POINTER(SoftKey), c_int32, c_int64, c_void_p, c_int32,
                                     c_void_p, c_void_p]),
    "tdp_soft_groupby_bwd": (c_int, [POINTER(SoftKey), c_int32, c_int64, c_void_p, c_int32,
                                     c_void_p, POINTER(c_void_p), c_void_p, c_void_p]),
    "tdp_linear_fwd": (c_int, [c_void_p, c_int32, c_int64, c_int32, c_int32, c_void_p, c_void_p,
                               c_void_p, c_void_p]),
    "tdp_linear_wgrad_workspace": (c_size_t, [c_int64, c_int32, c_int32]),
    "tdp_linear_wgrad": (c_int, [c_void_p, c_void_p, c_int32, c_int64, c_int32, c_int32, c_void_p,
                                 c_void_p, c_void_p, c_size_t, c_void_p]),
    "tdp_soft_linear_supported": (c_int, [c_int32, c_int64, c_int32, c_int32, c_int64, c_void_p]),
    "tdp_linear_argmax_count": (c_int, [c_void_p, c_int32, c_int64, c_int32, c_int32, c_void_p,
                                        c_void_p, POINTER(SoftKey), c_int32, c_int32, c_void_p,
                                        c_void_p]),
    "tdp_soft_linear_count_fwd": (c_int, [c_void_p, c_int32, c_int64, c_int32, c_int32, c_void_p,
                                          c_void_p, POINTER(SoftKey), c_int32, c_int32, c_void_p,
                                          c_void_p]),
    "tdp_soft_linear_count_bwd_workspace": (c_size_t, [c_int64, c_int32, c_int32]),
    "tdp_soft_linear_count_bwd": (c_int, [c_void_p, c_int32, c_int64, c_int32, c_int32, c_void_p,
                                          c_void_p, POINTER(SoftKey), c_int32, c_int32, c_void_p,
                                          c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
}

_lock = threading.Lock()
_lib: Optional[ctypes.CDLL] = None


def library_path() -> Path:
    return _LIB_PATH


def load() -> ctypes.CDLL:
    """Load libtdp_kernels.so (built in-tree by ``__graft_entry__.build()``)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise NativeError(
                    f"{_LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (the B200 kernels have no CPU fallback)")
            lib = ctypes.CDLL(str(_LIB_PATH))
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def last_error() -> str:
    msg = load().tdp_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> int:
    if rc < 0:
        raise NativeError(f"{what} failed ({rc}): {last_error()}")
    return rc


def call(name: str, *args) -> int:
    return check(getattr(load(), name)(*args), name)


# ---------------------------------------------------------------------------
# argument helpers
# ---------------------------------------------------------------------------

def require_cuda(*tensors: torch.Tensor) -> None:
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise NativeError(
                f"B200 kernels need CUDA tensors; got a {t.device} tensor (no CPU fallback)")


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_raw_device = getattr(torch._C, "_cuda_getDevice", None)


def stream() -> c_void_p:
    """The current CUDA stream of the current device (torch's raw accessors:
    this is called once per launch, torch.cuda.current_stream() costs ~10 us)."""
    if _raw_stream is not None and _raw_device is not None:
        return c_void_p(_raw_stream(_raw_device()))
    return c_void_p(torch.cuda.current_stream().cuda_stream)


def current_device() -> int:
    """torch.cuda.current_device() without its Python-level checks."""
    if _raw_device is not None:
        return int(_raw_device())
    return torch.cuda.current_device()


def ptr(t: Optional[torch.Tensor]) -> c_void_p:
    return c_void_p(0 if t is None else t.data_ptr())


def column(t: torch.Tensor, device_check: bool = True) -> Column:
    """Descriptor of a contiguous tensor.  ``device_check=False`` is only for
    the no-launch diagnostics (tdp_pipeline_codegen) on GPU-less hosts."""
    if device_check:
        require_cuda(t)
    if not t.is_contiguous():
        raise NativeError("column tensors must be contiguous")
    dt = TORCH_TO_TDP.get(t.dtype)
    if dt is None:
        raise NativeError(f"unsupported column dtype {t.dtype}")
    rows = t.shape[0] if t.dim() else 1
    width = 1
    for s in t.shape[1:]:
        width *= s
    return Column(c_void_p(t.data_ptr()), dt, 0, rows, width)


def columns(ts: Sequence[torch.Tensor], device_check: bool = True):
    arr = (Column * max(1, len(ts)))()
    for i, t in enumerate(ts):
        arr[i] = column(t, device_check)
    return arr


def struct_array(cls, items: Sequence):
    arr = (cls * max(1, len(items)))()
    for i, it in enumerate(items):
        arr[i] = it
    return arr


def workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)


def sm_count() -> int:
    return int(load().tdp_device_sm_count())


def launch_count() -> int:
    """Kernels launched by libtdp_kernels so far in this process."""
    return int(load().tdp_launch_count())

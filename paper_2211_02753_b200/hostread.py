"""Host reads of device-computed integers (row counts, group counts, key
ranges, validation flags), made replayable.

A plan whose output sizes depend on the data -- a join sizing its pair
buffers, a group-by sizing its groups -- synchronises with the device to
read those integers.  Over an unchanged catalog they are the same on every
run, so a CUDA-graph capture of the plan (replay.py) may take them from a
log written by an earlier eager run instead of synchronising:

* ``recording(log)``: every :func:`read_ints` reads the device as usual and
  appends the values to ``log``;
* ``replaying(log)`` (inside a graph capture): :func:`read_ints` returns the
  next logged values and enqueues ``tdp_expect_values``, a one-thread kernel
  that compares the device values with the logged ones on every replay and
  traps on a mismatch -- a catalog modified behind torch's version counters
  aborts the replay loudly instead of letting kernels write past buffers
  sized from stale counts.

Outside both contexts :func:`read_ints` is a plain synchronising read.
"""

from __future__ import annotations

import threading
from ctypes import c_int64
from typing import Optional

import torch

from . import _native as nat

_TLS = threading.local()

MAX_VALUES = 16  # per read (tdp_expect_values)


class ReplayMismatch(RuntimeError):
    """The read sequence of a capture run diverged from the recorded one."""


class _Log:
    """Python-side reads (``values``) and the library's own decisions
    (``c_values``: the radix sort's digit passes, logged in C)."""

    __slots__ = ("mode", "values", "pos", "c_values", "c_pos", "decisions", "d_pos")

    def __init__(self, mode: str, values: Optional[list] = None,
                 c_values: Optional[list] = None, decisions: Optional[list] = None):
        self.mode = mode
        self.values = [] if values is None else values
        self.pos = 0
        self.c_values = [] if c_values is None else c_values
        self.c_pos = 0
        self.decisions = [] if decisions is None else decisions
        self.d_pos = 0

    def consumed(self) -> bool:
        return (self.pos == len(self.values) and self.c_pos == len(self.c_values)
                and self.d_pos == len(self.decisions))


def active() -> bool:
    """A pipeline is being recorded or captured on this thread."""
    return getattr(_TLS, "log", None) is not None


class _Scope:
    def __init__(self, log: _Log):
        self.log = log

    def __enter__(self):
        if getattr(_TLS, "log", None) is not None:
            raise RuntimeError("nested host-read log scopes")
        log = self.log
        if log.mode == "record":
            nat.call("tdp_replay_log_begin", 1, None, 0)
        else:
            vals = (c_int64 * max(1, len(log.c_values)))(*log.c_values)
            nat.call("tdp_replay_log_begin", 2, vals, len(log.c_values))
        _TLS.log = log
        return log

    def __exit__(self, *exc):
        _TLS.log = None
        lib = nat.load()
        n = int(lib.tdp_replay_log_size())
        if self.log.mode == "record":
            buf = (c_int64 * max(1, n))()
            lib.tdp_replay_log_end(buf, n)
            self.log.c_values = [int(v) for v in buf[:n]]
        else:
            self.log.c_pos = n
            lib.tdp_replay_log_end(None, 0)
        return False


def recording() -> _Scope:
    return _Scope(_Log("record"))


def replaying(log: "_Log") -> _Scope:
    """A fresh replay cursor over a recorded log."""
    return _Scope(_Log("replay", log.values, log.c_values, log.decisions))


SYNC_READS = [0]  # synchronising reads of device integers in this process (diagnostics)


def _sync_read(t: torch.Tensor) -> list[int]:
    if t.is_cuda:
        SYNC_READS[0] += 1
    return [int(v) for v in t.reshape(-1).tolist()]


def read_ints(t: torch.Tensor) -> list[int]:
    """The integer elements of a small device tensor (int64 / int32 / bool)."""
    log = getattr(_TLS, "log", None)
    if log is None:
        return _sync_read(t)
    if log.mode == "record":
        vals = _sync_read(t)
        log.values.append(vals)
        return vals
    if log.pos >= len(log.values):
        raise ReplayMismatch("more host reads than recorded")
    vals = log.values[log.pos]
    log.pos += 1
    flat = t.reshape(-1)
    if flat.numel() != len(vals) or len(vals) > MAX_VALUES:
        raise ReplayMismatch("host read shape differs from the recorded one")
    if flat.dtype == torch.bool:
        flat = flat.to(torch.int32)
    esize = flat.element_size()
    if esize not in (4, 8) or flat.dtype.is_floating_point:
        raise ReplayMismatch(f"unsupported host read dtype {flat.dtype}")
    flat = flat.contiguous()
    expected = (c_int64 * MAX_VALUES)(*vals)
    nat.call("tdp_expect_values", nat.ptr(flat), esize, len(vals), expected, nat.stream())
    return list(vals)


def decision(fn):
    """A planning decision taken from host-side state (a cached column
    statistic): ``fn()`` normally and while recording (logged); inside a
    capture, the recorded decision -- so the captured plan takes the same
    path as the run it was recorded from even if that state is not available
    to it (statistics of a tensor created in the capture).  Device data the
    decision rests on is still checked by the kernels' own logged reads."""
    log = getattr(_TLS, "log", None)
    if log is None:
        return fn()
    if log.mode == "record":
        v = fn()
        log.decisions.append(v)
        return v
    if log.d_pos >= len(log.decisions):
        raise ReplayMismatch("more planning decisions than recorded")
    v = log.decisions[log.d_pos]
    log.d_pos += 1
    return v


def read_int(t: torch.Tensor) -> int:
    return read_ints(t)[0]


def replay_value(dev: torch.Tensor) -> Optional[int]:
    """Inside a replaying scope: the logged value of a deferred device count
    (checked on the device like :func:`read_ints`); None otherwise."""
    log = getattr(_TLS, "log", None)
    if log is None or log.mode != "replay":
        return None
    return read_ints(dev)[0]


def record_value(v: int) -> None:
    """Inside a recording scope: log a deferred count read through its pinned
    host slot (the capture reads it with :func:`replay_value`)."""
    log = getattr(_TLS, "log", None)
    if log is not None and log.mode == "record":
        log.values.append([int(v)])

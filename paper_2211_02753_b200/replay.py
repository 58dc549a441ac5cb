"""CUDA-graph replay of exact query plans over an unchanged catalog.

The reference re-interprets its operator program on every ``run``
(tq/compiler.py:366-367).  Here that interpretation is Python planning around
a handful of kernel launches (~0.3 ms for Q1), comparable to the launches
themselves once columns are narrow or shards small.  An exact query is a pure
function of the catalog state (SPEC plan-compiler: "run twice -> identical
results"), so ``CompiledQuery.run`` captures the plan's launches into a CUDA
graph the second time it sees the same state and replays it afterwards:

* state = the scanned tables (object identity, every stored column buffer and
  its in-place version counter), the UDF registry, the versions of the
  referenced parameters, the device and the process group of the enclosing
  ``distributed.sharded`` scope; anything else (a gloo group, an open tape,
  an unknown lazy column) disables replay;
* under NCCL the in-query collectives (the all-reduce of partial aggregates,
  the all-to-all of a key shuffle) are captured with the kernels: every rank
  captures on the same (second) run of the same plan and replays in lockstep;
* every kernel still runs over every row on each replay -- only the host-side
  planning is skipped -- and the launches are accounted to the library's
  launch counter;
* the result is a fresh table: the result buffers written by the graph are
  copied out of its memory pool, device row counts get fresh host slots.

A plan that cannot be captured (a host synchronisation inside, e.g. a join
sizing its output) runs eagerly from then on.  ``TDP_REPLAY=0`` or
``CompileConfig(replay=False)`` turn replay off.
"""

from __future__ import annotations

import ctypes
import gc
import os
import threading
import warnings
import weakref
from collections import OrderedDict
from typing import Optional

import torch

from . import _native as nat
import torch.distributed as dist

from .distributed import current_group
from .encodings import EncodedTensor, trusted
from . import hostread
from .lazy import DeferredCount, LazyValue, PrefixRows, capturing, compact_source
from .storage import Table, table_from_columns
from .tensor import Tensor, _cuda_available

MAX_ENTRIES = 4
MAX_RESULT_BYTES = 64 << 20  # larger results: the copy-out would dominate

_NOGRAPH = "nograph"


def enabled() -> bool:
    return os.environ.get("TDP_REPLAY", "1") != "0"


def _stored(t: Tensor) -> Optional[torch.Tensor]:
    """The buffer a catalog column's values live in, if plainly known."""
    if t._t is not None:
        return t._t
    lz = t._lazy
    if isinstance(lz, LazyValue) and lz.sel is None:
        if lz.expr.op == "col":
            return lz.expr.col
        src = compact_source(lz.expr)
        if src is not None:
            return src[0]
    return None


def _tables_signature(catalog, names) -> Optional[tuple[list, list]]:
    """(signature items, tables) of the named catalog tables: identity, every
    stored column buffer and its in-place version counter."""
    group = current_group()
    if group is not None and dist.get_backend(group) != "nccl":
        return None  # host-staged (gloo) collectives cannot be captured
    if not _cuda_available() or torch.cuda.is_current_stream_capturing() or hostread.active():
        return None
    tables_by_name = getattr(catalog, "_tables", None)
    if tables_by_name is None:
        return None
    # a sharded run (NCCL collectives inside the graph: capturable, replayed in
    # lockstep on every rank) and a local one are different states
    sig, tables = [id(catalog), nat.current_device(), id(group) if group else None], []
    for name in names:
        t = tables_by_name.get(name)
        if t is None:
            return None
        tables.append(t)
        sig.append(id(t))
        for c in t.columns:
            st = _stored(c.values)
            if st is None or not st.is_cuda:
                return None
            sig.append(st.data_ptr())
            sig.append(st._version)
    return sig, tables


def signature(q, catalog) -> Optional[tuple]:
    got = _tables_signature(catalog, q._scan_tables)
    if got is None:
        return None
    sig = got[0] + [id(q.registry), len(q.registry.names())]
    for p in q._params:
        d = p.value.data
        sig.append(d.data_ptr())
        sig.append(d._version)
    return tuple(sig)


class _Template:
    """Result table of a captured run and how to re-materialise it: the pool
    storages to copy out, and per result tensor a precomputed (storage,
    dtype, size, stride, offset) so the fresh table is built from strided
    views of the copies without re-deriving anything."""

    def __init__(self, schema, cols, storages, device, rows):
        self.schema = schema
        self.cols = cols          # ("t", spec, None, enc) | ("prefix", spec, count_spec, enc)
        self.storages = storages  # key -> uint8 view of a pool storage
        self.device = device
        self.rows = rows          # int row count of plain-tensor results, else None

    @staticmethod
    def build(table, inputs: set) -> Optional["_Template"]:
        cols, storages, total = [], {}, 0

        def track(t: torch.Tensor):
            """Spec of ``t`` (None: too much to copy out)."""
            nonlocal total
            st = t.untyped_storage()
            key = st.data_ptr()
            if key in inputs:
                return ("input", t)
            if key not in storages:
                total += st.nbytes()
                if total > MAX_RESULT_BYTES or st.nbytes() % t.element_size():
                    return None
                storages[key] = torch.empty(0, dtype=torch.uint8, device=t.device).set_(
                    st, 0, (st.nbytes(),), (1,))
            return (key, t.dtype, tuple(t.size()), tuple(t.stride()), t.storage_offset())

        rows = None
        for c in table.columns:
            v = c.values
            if v._t is not None:
                spec = track(v._t)
                if spec is None:
                    return None
                cols.append(("t", spec, None, c.encoding))
                rows = int(v._t.shape[0]) if v._t.dim() else None
            elif isinstance(v._lazy, PrefixRows) and isinstance(v._lazy.count, DeferredCount) \
                    and v._lazy.count.dev is not None:
                fs, ds = track(v._lazy.full), track(v._lazy.count.dev)
                if fs is None or ds is None:
                    return None
                cols.append(("prefix", fs, ds, c.encoding))
            else:
                return None
        if any(kind == "prefix" for kind, *_ in cols):
            rows = None
        return _Template(table.schema, cols, storages, table.device, rows)

    def materialise(self):
        fresh = {k: src.clone() for k, src in self.storages.items()}
        typed: dict = {}

        def view(spec) -> torch.Tensor:
            if spec[0] == "input":  # a catalog buffer passed through
                return spec[1]
            key, dt, size, stride, off = spec
            base = typed.get((key, dt))
            if base is None:
                base = fresh[key].view(dt)
                typed[(key, dt)] = base
            return base.as_strided(size, stride, off)

        cols = []
        count = None
        with trusted():
            for kind, a, b, enc in self.cols:
                if kind == "t":
                    cols.append(EncodedTensor(Tensor(view(a)), enc))
                else:
                    if count is None or count[0] != b:  # one host slot per device count
                        count = (b, DeferredCount(view(b)))
                    cols.append(EncodedTensor(Tensor(PrefixRows(view(a), count[1])), enc))
        if self.rows is None and count is None:
            return table_from_columns(list(self.schema.names), cols, device=self.device)
        return Table(self.schema, tuple(cols), count[1] if count is not None else self.rows,
                     self.device)


class _Replay:
    """A captured plan.  Replays are serialised: exact runs may come from
    several threads on different streams (SPEC: read-only runs may proceed in
    parallel), and every replay rewrites the graph's buffers, so a replay
    first waits (on the device) for the previous replay's copy-out."""

    def __init__(self, graph, template: _Template, launches: int, hold):
        self.graph = graph
        self.template = template
        self.launches = launches
        self.hold = hold  # the catalog tables the signature names (ids stay unique)
        self.lock = threading.Lock()
        # one event, re-recorded after every copy-out; a replay from another
        # stream waits on it (same stream: stream order already serialises)
        self.done = torch.cuda.Event()
        self.done.record()  # creates the event (torch creates it lazily)
        self.done_handle = ctypes.c_void_p(self.done.cuda_event)
        self.last_stream: Optional[int] = None

    def __call__(self):
        with self.lock:
            lib = nat.load()
            st = nat.stream()
            if self.last_stream is not None and self.last_stream != st.value:
                nat.check(lib.tdp_stream_wait_event(st, self.done_handle), "tdp_stream_wait_event")
            self.graph.replay()
            table = self.template.materialise()
            nat.check(lib.tdp_replay_done(self.done_handle, st, self.launches), "tdp_replay_done")
            self.last_stream = st.value
            return table


def _inputs(tables) -> set:
    ptrs = set()
    for t in tables:
        for c in t.columns:
            st = _stored(c.values)
            if st is not None:
                ptrs.add(st.untyped_storage().data_ptr())
    return ptrs


CAPTURES = [0]  # capture attempts in this process (diagnostics)
CAPTURE_ATTEMPTS = 2  # failed captures of one state before it runs eagerly for good


def _capture(execute, tables, log):
    """Capture ``execute`` into a CUDA graph; its host reads of device
    integers come from ``log`` (an eager run over the same state) and are
    checked on the device on every replay (hostread.py)."""
    CAPTURES[0] += 1
    inputs = _inputs(tables)
    torch.cuda.synchronize()
    # a stale (non-sticky) error left by an unrelated earlier call would make
    # the first launch check inside the capture fail it
    nat.load().tdp_clear_error()
    graph = torch.cuda.CUDAGraph()
    launches0 = nat.launch_count()
    # no cyclic garbage collection inside the capture: a collected object of an
    # earlier run holding a CUDA event (a DeferredCount) would destroy it, an
    # API call that invalidates the capture
    gc_was_enabled = gc.isenabled()
    gc.disable()
    try:
        with capturing(), warnings.catch_warnings(), hostread.replaying(log) as rlog:
            warnings.simplefilter("ignore")  # "graph is empty": a lazy result, no launches
            # thread_local: an eager query on another thread (or NCCL's
            # watchdog polling its events) does not invalidate this capture
            with torch.cuda.graph(graph, capture_error_mode="thread_local"):
                table = execute()
        if not rlog.consumed():
            raise hostread.ReplayMismatch("fewer host reads than recorded")
    except Exception:
        if gc_was_enabled:
            gc.enable()
        # an uncapturable call inside the plan (or a diverging read sequence)
        if os.environ.get("TDP_REPLAY_DEBUG"):
            import traceback

            traceback.print_exc()
        nat.load().tdp_clear_error()
        torch.cuda.synchronize()
        return _NOGRAPH
    if gc_was_enabled:
        gc.enable()
    launches = nat.launch_count() - launches0
    template = _Template.build(table, inputs)
    if template is None:
        return _NOGRAPH
    return _Replay(graph, template, launches, list(tables))


class _Warm:
    """First sighting of a state: weak references to its tables, so a second
    sighting is recognised only while those very objects are alive (a new
    table that happens to reuse a dead one's id and buffers is a new state,
    and a stream of fresh tables never triggers captures), and the host reads
    the eager run made (None until it finished)."""

    def __init__(self, tables):
        self.refs = [weakref.ref(t) for t in tables]
        self.log = None  # hostread._Log
        self.failures = 0

    def alive(self, tables) -> bool:
        return all(r() is t for r, t in zip(self.refs, tables))


_LOCK = threading.Lock()  # the per-owner replay tables


def run(owner, sig, tables, execute):
    """Result of ``execute()`` (a Table) for the state ``sig``: replayed from
    a CUDA graph once the state has been seen before, else run eagerly (the
    first eager run records its host reads for the capture).  ``owner`` keeps
    the entries (``owner._replays``, an OrderedDict)."""
    with _LOCK:
        ent = _lookup(owner, sig, tables, execute)
    if isinstance(ent, _Replay):
        return ent()
    if isinstance(ent, _Warm):
        with hostread.recording() as log:
            out = execute()
        ent.log = log
        return out
    return execute()


def _lookup(owner, sig, tables, execute):
    entries: OrderedDict = owner._replays
    ent = entries.get(sig)
    if ent is None or (isinstance(ent, _Warm) and not ent.alive(tables)):
        ent = _Warm(tables)
        entries[sig] = ent
        entries.move_to_end(sig)
        while len(entries) > MAX_ENTRIES:
            entries.popitem(last=False)
        return ent
    if ent == _NOGRAPH:
        return None
    if isinstance(ent, _Warm):
        if ent.log is None:  # no finished recording (another thread's, or one that raised)
            return ent
        got = _capture(execute, tables, ent.log)
        if got == _NOGRAPH:
            # one more attempt on the next sighting (a one-time lazy
            # initialisation inside the first capture can abort it), then eager
            ent.failures += 1
            if ent.failures >= CAPTURE_ATTEMPTS:
                entries[sig] = _NOGRAPH
            return None
        ent = got
        entries[sig] = ent
    entries.move_to_end(sig)
    return ent


class Pipeline:
    """Replay for a composite plan -- several compiled queries and kernel
    calls between them, ``fn(catalog) -> Table`` over the catalog tables
    ``table_names`` -- on the same terms as ``CompiledQuery.run``: an
    unchanged state replays one CUDA graph of the whole plan, its data-
    dependent sizes (join pair counts, group counts) taken from the recorded
    eager run and checked on the device."""

    def __init__(self, fn, table_names):
        self.fn = fn
        self.table_names = tuple(table_names)
        self._replays: OrderedDict = OrderedDict()

    def run(self, catalog):
        if not enabled():
            return self.fn(catalog)
        got = _tables_signature(catalog, self.table_names)
        if got is None:
            return self.fn(catalog)
        sig, tables = got
        return run(self, tuple(sig), tables, lambda: self.fn(catalog))

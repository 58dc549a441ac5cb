"""TPC-H Q1 / Q6 on lineitem (BASELINE configs 1-2): the headline bench line.

Layout: the synthetic SF lineitem table is split into N contiguous row
ranges (``distributed.shard_bounds``), one per rank ("strong" scaling, the
BASELINE row-sharded config); ``--scaling weak`` gives every rank an SF-sized
range of an SF x N table instead.  A step is ``CompiledQuery.run(catalog)``
of the Appendix-A SQL plan inside ``distributed.sharded()``: the fused scan
over the local rows, the NCCL all-reduce of the partial aggregates, the
finalisation -- replayed as one CUDA graph over an unchanged catalog.
"""

from __future__ import annotations

import json
import os
import time

from .common import (ROOT, ClockSampler, barrier, cpu_model, dist_env, host_cores, init_dist,
                     max_over_ranks, peaks, sum_over_ranks, sustain, timed)

METRIC = "TPC-H Q1/Q6 SF10 rows/sec & HBM GB/s at 1/2/4/8 B200 vs CPU ref"
Q6_COLS = ("l_shipdate", "l_quantity", "l_extendedprice", "l_discount")


def table_layout(args, world: int, rank: int) -> tuple[float, int, int, int]:
    """(table SF, table rows, this rank's [lo, hi))."""
    from paper_2211_02753_b200.distributed import shard_bounds

    if args.scaling == "weak":
        per = int(round(6_000_000 * args.sf))
        return args.sf * world, per * world, rank * per, (rank + 1) * per
    n = int(round(6_000_000 * args.sf))
    lo, hi = shard_bounds(n, rank, world)
    return args.sf, n, lo, hi


def config(args, world: int) -> dict:
    """The workload description, identical in both arms (``same_config``)."""
    sf_table, n, _, _ = table_layout(args, world, 0)
    if args.query == "q1":
        w = {"workload": f"TPC-H Q1 SF{sf_table:g}: filter l_shipdate<=10471 -> q1prep UDF "
                         "(disc_price, charge) -> GROUP BY returnflag, linestatus, 8 aggregates",
             "bytes_per_row": 56,
             "columns": "7 x 8 B (int64 dates/dictionary codes, float64 values)"}
    else:
        w = {"workload": f"TPC-H Q6 SF{sf_table:g}: 5-predicate filter -> revenue UDF -> SUM",
             "bytes_per_row": 32, "columns": "4 x 8 B (int64 shipdate, float64 values)"}
    w.update(sf=sf_table, rows=n, scaling=args.scaling, encoding=args.encoding,
             parallelism=(f"dp{world}: {world} contiguous row shards of one SF{sf_table:g} table "
                          f"(strong)" if args.scaling == "strong" else
                          f"dp{world}: one SF{args.sf:g} row shard per rank (weak)"),
             l2="inputs larger than L2 (no flush needed)" if n * w["bytes_per_row"] / world > 4e8
             else "inputs smaller than 3x L2: every step re-reads HBM (no flush)",
             data="synthetic, seeded dbgen-like lineitem (SURVEY Appendix B, "
                  "workloads.lineitem_arrays seed 42)")
    if args.encoding == "compact":
        w["columns"] = ("compact storage (SURVEY §8(f) 1): int16 dates, uint8 dictionary codes, "
                        "scaled-decimal int8/int32 values; decoded values bit-identical to the "
                        "8 B reference columns")
    return w


# ---------------------------------------------------------------------------
# full-table oracle (parity of the timed result) -- test infrastructure
# ---------------------------------------------------------------------------

_PARITY_POOL = None


def start_parity_pool(processes: int):
    """Worker processes for the oracle, forked before CUDA is initialised."""
    global _PARITY_POOL
    import multiprocessing as mp

    _PARITY_POOL = mp.get_context("fork").Pool(processes)
    return _PARITY_POOL


def _oracle_chunk(task):
    from oracle import tpch as otpch
    from paper_2211_02753_b200 import workloads as wl

    query, sf, n, lo, hi = task
    a = wl.lineitem_arrays(sf, 42, rows=n, lo=lo, hi=hi)
    return otpch.q1_partial(a) if query == "q1" else otpch.q6_partial(a)


def full_oracle(query: str, sf: float, n: int) -> dict:
    """The oracle's result over all ``n`` rows of the table (every shard),
    computed chunk-parallel on the host cores and merged."""
    from oracle import tpch as otpch
    from paper_2211_02753_b200.workloads import LINEITEM_CHUNK

    tasks = [(query, sf, n, lo, min(n, lo + LINEITEM_CHUNK)) for lo in range(0, n, LINEITEM_CHUNK)]
    parts = _PARITY_POOL.map(_oracle_chunk, tasks) if _PARITY_POOL else list(map(_oracle_chunk, tasks))
    return otpch.q1_merge(parts) if query == "q1" else otpch.q6_merge(parts)


def check(result, exp: dict) -> tuple[bool, dict]:
    """Keys / counts bit-exact, float aggregates rtol 1e-9 (stated bound 1e-5)."""
    import numpy as np

    got = {n: c.values.numpy() for n, c in zip(result.schema.names, result.columns)}
    ok, worst = True, 0.0
    for k, v in exp.items():
        g = got[k]
        if v.dtype.kind in "iu":
            ok &= bool(g.shape == v.shape and np.array_equal(g, v))
        else:
            ok &= bool(g.shape == v.shape and np.allclose(g, v, rtol=1e-9, atol=0))
            if g.shape == v.shape and len(v):
                worst = max(worst, float(np.max(np.abs(g - v) / np.maximum(np.abs(v), 1e-300))))
    return ok, {"max_rel_err": worst}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args) -> None:
    world, rank, local = dist_env()
    parity = rank == 0 and not args.no_parity
    if parity:
        start_parity_pool(min(16, host_cores()))
    import torch

    group = init_dist(world, local)
    import paper_2211_02753_b200 as tq
    from paper_2211_02753_b200 import _native, hostread, workloads as wl
    from paper_2211_02753_b200.distributed import sharded

    sf_table, n_total, lo, hi = table_layout(args, world, rank)
    rows = hi - lo
    arrays = wl.lineitem_arrays(sf_table, 42, rows=n_total, lo=lo, hi=hi)
    if args.query == "q1":
        sql, reg, cols = wl.Q1_SQL, wl.q1_registry(), wl.LINEITEM_COLUMNS
    else:
        sql, reg, cols = wl.Q6_SQL, wl.q6_registry(), Q6_COLS
    bpr = config(args, world)["bytes_per_row"]
    table = wl.lineitem_table(arrays, cols)
    stored_bpr = bpr
    if args.encoding == "compact":  # ingestion, outside the timed region
        from paper_2211_02753_b200 import compact as cp

        table = cp.compact_table(table)
        stored_bpr = sum(cp.stored_bytes(c) for c in table.columns)
    cat = tq.Catalog()
    cat.register("lineitem", table)
    query = wl.compile_sql(sql, cat, reg)
    lib = _native.load()
    import ctypes as ct

    def kernel_timer(fn, steps):
        """Mean library-event time of the fused scan kernel over eager runs
        (a replayed graph cannot record the library's events) and the eager
        step time (the plan re-run on the host each step)."""
        os.environ["TDP_REPLAY"] = "0"
        try:
            eager = timed(fn, steps, group)
            lib.tdp_kernel_timer_enable(1)
            lib.tdp_kernel_timer_read(None, None)
            timed(fn, steps, group)
            lib.tdp_kernel_timer_enable(0)
        finally:
            os.environ.pop("TDP_REPLAY", None)
        tot, cnt = ct.c_double(0.0), ct.c_int64(0)
        lib.tdp_kernel_timer_read(ct.byref(tot), ct.byref(cnt))
        k = tot.value / cnt.value if cnt.value else 0.0
        k, eager = max_over_ranks([k, eager], group)
        return k, eager

    with sharded(group):
        holder = {}

        def step():
            holder["r"] = query.run(cat)

        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        sampler = ClockSampler(local)
        launches0 = _native.launch_count()
        reads0 = hostread.SYNC_READS[0]
        sampler.active = True
        ms = timed(step, args.steps, group)
        launches = _native.launch_count() - launches0
        sync_reads = hostread.SYNC_READS[0] - reads0
        timed_result = holder["r"]  # the last timed (replayed) step's output
        # clocks: keep the GPU loaded for >= 1.5 s so nvidia-smi samples it
        barrier(group)
        sustain(step, 1.5)
        barrier(group)
        clocks = sampler.stop()
        launches = sum_over_ranks(launches, group)
        kernel_ms, eager_ms = kernel_timer(step, args.steps)

        companion = None
        if args.query == "q1" and not args.no_companion:
            q6 = wl.compile_sql(wl.Q6_SQL, cat, wl.q6_registry())
            h6 = {}

            def step6():
                h6["r"] = q6.run(cat)

            for _ in range(3):
                step6()
            ms6 = timed(step6, args.steps, group)
            r6 = h6["r"]
            k6, eager6 = kernel_timer(step6, args.steps)
            companion = {"workload": f"TPC-H Q6 SF{sf_table:g} on the same lineitem shards",
                         "value": n_total / (ms6 / 1e3), "unit": "rows/s", "ms_per_step": ms6,
                         "eager_ms_per_step": eager6, "kernel_ms": k6}
            if args.encoding == "wide" and k6:
                companion["hbm_gbs_kernel"] = 32 * rows / (k6 / 1e3) / 1e9
                companion["peak_frac_kernel"] = companion["hbm_gbs_kernel"] / peaks()[0]

        # ---- end to end through the API from pinned host buffers ----------
        if args.encoding == "compact":
            from paper_2211_02753_b200 import compact as cp

            host_stored = [t.cpu().pin_memory() for t in cp.stored_tensors(table)]
            h2d = sum(h.numel() * h.element_size() for h in host_stored)

            def make_table():
                return cp.table_from_stored(table, [h.to("cuda", non_blocking=True)
                                                    for h in host_stored])
        else:
            host = {c: torch.from_numpy(arrays[c]).pin_memory() for c in cols}
            h2d = sum(h.numel() * h.element_size() for h in host.values())

            def make_table():
                return wl.lineitem_table(host, cols)

        d2h = [0]

        def e2e_step():
            c2 = tq.Catalog()
            c2.register("lineitem", make_table())
            out = query.run(c2)
            d2h[0] = sum(c.values.numpy().nbytes for c in out.columns)

        e2e_step()
        barrier(group)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        barrier(group)
        e2e_s = max_over_ranks([(time.perf_counter() - w0) / args.e2e_steps], group)[0]
        h2d_total = sum_over_ranks(h2d, group)

    # ---- parity of the TIMED outputs against the oracle over the whole table
    par = None
    if parity:
        w0 = time.perf_counter()
        exp = full_oracle(args.query, sf_table, n_total)
        ok, detail = check(timed_result, exp)
        par = {"status": "ok" if ok else "MISMATCH", "rows": n_total,
               "checked": "the last timed (CUDA-graph replayed) step's result table",
               "rule": "keys/counts bit-exact, float aggregates rtol 1e-9 vs the float64 oracle "
                       "(stated bound 1e-5)", "oracle_s": time.perf_counter() - w0, **detail}
        if companion is not None:
            ok6, d6 = check(r6, full_oracle("q6", sf_table, n_total))
            companion["parity"] = {"status": "ok" if ok6 else "MISMATCH", "rows": n_total, **d6}
    if rank != 0:
        _finish(group)
        return
    peak, peak_src = peaks()
    achieved = stored_bpr * rows / (kernel_ms / 1e3) / 1e9 if kernel_ms else None
    line = {
        "metric": METRIC,
        "value": n_total / (ms / 1e3),
        "unit": "rows/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": ms,
        "eager_ms_per_step": eager_ms,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded dbgen-like lineitem, SURVEY Appendix B), resident in HBM",
        "config": config(args, world),
        "step": "CompiledQuery.run(catalog) of the SQL plan inside distributed.sharded(): fused "
                "scan of the local shard + NCCL all-reduce of partials + finalise, replayed as one "
                "CUDA graph over the unchanged catalog; eager_ms_per_step = the same plan re-run "
                "on the host every step",
        "hbm_gbs_step": bpr * n_total / (ms / 1e3) / 1e9,
        "e2e": {"value": n_total / e2e_s, "unit": "rows/s", "h2d_bytes_per_step": h2d_total,
                "d2h_bytes_per_step": d2h[0], "h2d_gbs_per_rank": h2d / e2e_s / 1e9,
                "how": "pinned host columns -> device table -> CompiledQuery.run (a new catalog: "
                       "re-planned) -> result to host (bound by the host->device link)"},
        "gpu_launches": launches,
        "host_sync_reads_in_timed_region": sync_reads,
        "roofline": {"bound": "hbm", "kernel": "tdp_scan_agg (fused filter+UDF+group-by), per rank, "
                                               "timed by library CUDA events on its launch stream",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None,
                     "traffic": _traffic(args, rows), "traffic_source":
                         "profiles/roofline_traffic.json (ncu dram__bytes_read+write of one launch "
                         "at these rows per launch; null if not captured)",
                     "peak_source": peak_src, "kernel_ms": kernel_ms,
                     "algorithmic_bytes_per_launch": stored_bpr * rows,
                     "bytes_per_row": stored_bpr},
        "clocks": clocks,
        "parity": par,
    }
    if companion is not None:
        line["companion_q6"] = companion
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, arrays)
    print(json.dumps(line), flush=True)
    _finish(group)


def _finish(group):
    if group is not None:
        import torch.distributed as dist

        dist.destroy_process_group()


def _traffic(args, rows: int):
    tf = ROOT / "profiles" / "roofline_traffic.json"
    try:
        tj = json.loads(tf.read_text())
    except Exception:
        return None
    sfx = "_compact" if args.encoding == "compact" else ""
    ent = tj.get(f"{args.query}_rows{rows}{sfx}")
    if ent is None and rows == int(round(6_000_000 * args.sf)):
        ent = tj.get(f"{args.query}_sf{args.sf:g}_n1{sfx}")
    return ent


def cpu_baseline(args, arrays) -> dict:
    """The oracle (numpy restatement of the reference path) on ONE host core
    over a bounded sample of the same table (first SF1 of the shard)."""
    from oracle import tpch as otpch

    sample_rows = min(len(arrays["l_shipdate"]), 6_000_000)
    sample = {k: v[:sample_rows] for k, v in arrays.items()}
    fn = otpch.q1 if args.query == "q1" else otpch.q6
    reps, t = 0, 0.0
    while t < 10.0 and reps < 20:
        w0 = time.perf_counter()
        fn(sample)
        t += time.perf_counter() - w0
        reps += 1
    return {"value": reps * sample_rows / t, "unit": "rows/s", "cores": 1, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{sample_rows} rows (first SF{sample_rows / 6e6:g} of the table) x {reps} "
                      f"repetitions, oracle/tpch.py (numpy restatement of tq filter_exact -> "
                      f"UDF -> groupby_exact; calibrated against the reference in BASELINE.md)"}


# ---------------------------------------------------------------------------
# reference arm: the reference algorithm on all host cores
# ---------------------------------------------------------------------------

_REF_ARRAYS: dict = {}


def _ref_worker(task):
    from oracle import tpch as otpch

    query, lo, hi = task
    a = {k: v[lo:hi] for k, v in _REF_ARRAYS.items()}
    return otpch.q1_partial(a) if query == "q1" else otpch.q6_partial(a)


def run_reference(args) -> None:
    import multiprocessing as mp

    from oracle import tpch as otpch
    from paper_2211_02753_b200 import workloads as wl

    world, rank, _ = dist_env()
    if rank != 0:
        return
    cores = host_cores()
    sf_table, n_total, _, _ = table_layout(args, world, 0)
    # calibrate one core, then size the per-step sample so the run stays short
    cal = wl.lineitem_arrays(sf_table, 42, rows=n_total, lo=0, hi=min(n_total, 1_000_000))
    _REF_ARRAYS.clear()
    _REF_ARRAYS.update(cal)
    w0 = time.perf_counter()
    _ref_worker((args.query, 0, len(cal["l_shipdate"])))
    per_core = len(cal["l_shipdate"]) / (time.perf_counter() - w0)
    budget_s = max(0.05, 150.0 / max(1, args.steps + args.warmup))
    sample = int(min(n_total, per_core * cores * budget_s))
    sample = max(sample, cores)
    arrays = wl.lineitem_arrays(sf_table, 42, rows=n_total, lo=0, hi=sample)
    _REF_ARRAYS.clear()
    _REF_ARRAYS.update(arrays)
    bounds = [(args.query, i * sample // cores, (i + 1) * sample // cores) for i in range(cores)]
    merge = otpch.q1_merge if args.query == "q1" else otpch.q6_merge
    with mp.get_context("fork").Pool(cores) as pool:
        for _ in range(args.warmup):
            merge(pool.map(_ref_worker, bounds))
        times = []
        for _ in range(args.steps):
            w0 = time.perf_counter()
            merge(pool.map(_ref_worker, bounds))
            times.append(time.perf_counter() - w0)
    step_s = sum(times) / len(times)
    value = sample / step_s
    line = {
        "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded dbgen-like lineitem, SURVEY Appendix B), in host RAM",
        "config": config(args, world),
        "impl": "reference",
        "arm": f"{cores} host processes over row ranges of the same table, partials merged "
               f"(oracle/tpch.py q1_partial/q1_merge); each step a {sample}-row sample",
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{sample} rows per step (first rows of the table), oracle/ "
                                   f"numpy restatement of the reference path on {cores} processes"},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)

"""Achieved HBM bandwidth of each relational operator at scale (the
north_star asks that every kernel's choice be evidenced by its achieved GB/s):
each operator runs through the package API on 6e7-row inputs, its CUDA
kernels' device time is summed from torch.profiler (host gaps excluded), and
the operator's algorithmic bytes (inputs read once + outputs written once)
are divided by it.  Prints one JSON line per operator.  Diagnostic tool, run
on the GPU box: python tools/kernel_zoo.py [rows]"""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200 import kernels as K
from paper_2211_02753_b200.autograd import gather_rows_raw

PEAK = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())[
    "hbm_gbs"] if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else 6537.0


def device_ms(fn, reps: int = 3) -> float:
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    total = 0.0
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            total += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    return total / reps / 1e3


def report(name: str, ms: float, nbytes: float, what: str):
    gbs = nbytes / (ms / 1e3) / 1e9
    print(json.dumps({"op": name, "device_ms": round(ms, 4), "algorithmic_bytes": nbytes,
                      "achieved_gbs": round(gbs, 1), "frac_of_copy_peak": round(gbs / PEAK, 3),
                      "bytes": what}), flush=True)


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 60_000_000
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(0)
    i64 = torch.randint(0, 1000, (n,), generator=g, device="cuda")
    f64 = torch.rand(n, generator=g, device="cuda", dtype=torch.float64)
    col_i, col_f = tq.plain(tq.Tensor(i64)), tq.plain(tq.Tensor(f64))

    # filter: comparison mask (8 B read + 1 B written per row)
    report("comparison_mask (tdp_filter_mask)", device_ms(lambda: K.comparison_mask(col_i, "<", 500)),
           9.0 * n, "8 B key read + 1 B mask written per row")
    # filter + compaction: indices of the passing rows (8 B read + 8 B per kept row)
    sel = (i64 < 300)
    m = int(sel.sum())

    def select():
        out = K.filter_exact([col_i], [(0, "<", 300)])
        out[0].values.data  # materialise the compacted column (indices + gather)
    report("filter_exact + materialise (tdp_filter_select, gather)", device_ms(select),
           8.0 * n + 8.0 * m + 16.0 * m, "8 B key per row + kept rows: 8 B index, 8 B read, 8 B write")
    # gather of a float column by a random permutation (index + value read, value written)
    perm = torch.randperm(n, generator=g, device="cuda")
    report("gather_rows (tdp_gather_rows)", device_ms(lambda: gather_rows_raw(f64, perm)), 24.0 * n,
           "8 B index + 8 B value read + 8 B written per row")
    # stable sort of an int64 column (values in [0, 1000): 2 digit passes)
    report("stable_order (tdp_sort_order, LSD radix)", device_ms(lambda: K.stable_order(col_i)),
           16.0 * n, "8 B key read + 8 B row index written (passes: extra)")
    # top-k of a float column
    report("topk_order k=10 (tdp_topk_order)", device_ms(lambda: K.topk_order(col_f, 10, True)),
           8.0 * n, "8 B key read per row")
    # hash group-by: 1e6 distinct sparse keys, SUM(f64) + COUNT
    keys = torch.randint(0, 1_000_000, (n,), generator=g, device="cuda") * 1_000_003 + 7
    kcol = tq.plain(tq.Tensor(keys))
    report("groupby_exact hash (1e6 sparse keys, SUM+COUNT)",
           device_ms(lambda: K.groupby_exact([kcol], [("sum", tq.Tensor(f64)), ("count", None)])),
           16.0 * n, "8 B key + 8 B value read per row (1e6 groups written: small)")
    # bitmap-rank group-by: 1e6 keys over a 5e6 range
    kb = torch.randint(0, 5_000_000, (n,), generator=g, device="cuda")
    kbcol = tq.plain(tq.Tensor(kb))
    report("groupby_exact bitmap rank (5e6 range, SUM+COUNT)",
           device_ms(lambda: K.groupby_exact([kbcol], [("sum", tq.Tensor(f64)), ("count", None)])),
           16.0 * n, "8 B key + 8 B value read per row")
    # sorted-runs group-by: a clustered key (runs of 1-7 rows)
    runs = torch.repeat_interleave(torch.arange(n, device="cuda"),
                                   torch.randint(1, 8, (n,), generator=g, device="cuda"))[:n]
    rcol = tq.plain(tq.Tensor(runs.contiguous()))
    ng = int(runs[-1]) + 1
    report("groupby_exact sorted runs (clustered key, SUM+COUNT)",
           device_ms(lambda: K.groupby_exact([rcol], [("sum", tq.Tensor(f64)), ("count", None)])),
           16.0 * n + 24.0 * ng, "8 B key + 8 B value read per row, key/count/sum per group")
    # joins: 1.5e7 unique build keys, 6e7 probe rows
    nb = n // 4
    build = torch.randperm(4 * nb, generator=g, device="cuda")[:nb]
    probe = torch.randint(0, 4 * nb, (n,), generator=g, device="cuda")
    for algo, rng_ in (("dense bitmap", (0, 4 * nb - 1)), ("hash", None)):
        K.JOIN_ALGORITHM = "auto"
        report(f"join_indices {algo} (1.5e7 build, 6e7 probe)",
               device_ms(lambda: K.join_indices(probe, build, build_range=rng_)),
               8.0 * nb + 8.0 * n, "8 B build key + 8 B probe key read (pairs written: extra)")
    K.JOIN_ALGORITHM = "sort"
    report("join_indices sort/searchsorted (1.5e7 build, 6e7 probe)",
           device_ms(lambda: K.join_indices(probe, build)), 8.0 * nb + 8.0 * n,
           "8 B build key + 8 B probe key read (pairs written: extra)")
    K.JOIN_ALGORITHM = "auto"


if __name__ == "__main__":
    main()

"""Host cost of a replayed CompiledQuery.run (Q6 SF1 by default): device time
per step vs host time per step, then a cProfile of the replay path.
Diagnostic only: python tools/profile_replay_host.py [q6|q1] [sf]"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200 import workloads as wl
from paper_2211_02753_b200.distributed import sharded

q = sys.argv[1] if len(sys.argv) > 1 else "q6"
sf = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cols = wl.LINEITEM_COLUMNS if q == "q1" else ("l_shipdate", "l_quantity", "l_extendedprice",
                                              "l_discount")
arrays = wl.lineitem_arrays(sf, 42, rows=int(6e6 * sf))
cat = tq.Catalog()
cat.register("lineitem", wl.lineitem_table(arrays, cols))
sql, reg = (wl.Q1_SQL, wl.q1_registry()) if q == "q1" else (wl.Q6_SQL, wl.q6_registry())
query = wl.compile_sql(sql, cat, reg)
with sharded(None):
    for _ in range(20):
        query.run(cat)
    torch.cuda.synchronize()
    N = 300
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(N):
        query.run(cat)
    e1.record()
    host_us = 1e6 * (time.perf_counter() - t0) / N
    torch.cuda.synchronize()
    print(f"{q} sf{sf}: device {1e3 * e0.elapsed_time(e1) / N:.1f} us/step, host enqueue "
          f"{host_us:.1f} us/step")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(300):
        query.run(cat)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(22)

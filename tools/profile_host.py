"""Host-side overhead of CompiledQuery.run on a tiny table (GPU time ~0)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200 import workloads as wl

q = sys.argv[1] if len(sys.argv) > 1 else "q1"
arrays = wl.lineitem_arrays(0.001, rows=4096)
cat = tq.Catalog()
cat.register("lineitem", wl.lineitem_table(arrays))
sql, reg = (wl.Q1_SQL, wl.q1_registry()) if q == "q1" else (wl.Q6_SQL, wl.q6_registry())
query = wl.compile_sql(sql, cat, reg)
for _ in range(20):
    query.run(cat)
torch.cuda.synchronize()
t0 = time.perf_counter()
N = 500
for _ in range(N):
    query.run(cat)
torch.cuda.synchronize()
print(f"{q}: {1e6 * (time.perf_counter() - t0) / N:.1f} us per run (host-bound)")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    query.run(cat)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

"""Eager (re-planned) Q3 step time after pipeline replays; capture counts."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2211_02753_b200 import replay, workloads as wl

tables = wl.q3_arrays(10.0, seed=7)
cat = wl.q3_catalog(tables)
plan = wl.Q3Plan(cat)
for name, fn in (("run (pipeline replay)", plan.run), ("run_eager", plan.run_eager)):
    for _ in range(3):
        fn(cat)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        fn(cat)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{name}: " + " ".join(f"{t:.2f}" for t in ts) + f"; captures so far {replay.CAPTURES[0]}")
print("tail entries:", [type(e).__name__ if not isinstance(e, str) else e for e in plan.tail._replays.values()])
for q in (plan.cust, plan.orders, plan.lineitem):
    print("filter entries:", [type(e).__name__ if not isinstance(e, str) else e for e in q._replays.values()])

"""Eager (re-planned) Q3 step time with and without replay of the inner queries."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2211_02753_b200 import replay, workloads as wl

tables = wl.q3_arrays(10.0, seed=7)
cat = wl.q3_catalog(tables)
plan = wl.Q3Plan(cat)
for name, fn in (("run_eager", plan.run_eager), ("run (pipeline replay)", plan.run)):
    for _ in range(3):
        fn(cat)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        fn(cat)
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms; captures so far {replay.CAPTURES[0]}")

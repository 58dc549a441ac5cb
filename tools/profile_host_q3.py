"""Host-side profile of the Q3-style pipeline (cProfile; diagnostic only)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2211_02753_b200 import workloads as wl

sf = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
eager = len(sys.argv) > 2 and sys.argv[2] == "eager"  # re-planned every run (no replay)
tables = wl.q3_arrays(sf, seed=7)
cat = wl.q3_catalog(tables)
plan = wl.Q3Plan(cat)
run = plan.run_eager if eager else plan.run
for _ in range(3):
    run(cat)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
for _ in range(20):
    run(cat)
torch.cuda.synchronize()
pr.disable()
print(f"{(time.perf_counter() - t0) / 20 * 1e3:.3f} ms per run (under cProfile)")
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)

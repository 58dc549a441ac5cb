import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2211_02753_b200 import workloads as wl, replay
from oracle import tpch as otpch
tables = wl.q3_arrays(0.02, seed=7)
cat = wl.q3_catalog(tables)
plan = wl.Q3Plan(cat)
for i in range(4):
    plan.run(cat)
    print(i, [type(e).__name__ for e in plan._pipeline._replays.values()], flush=True)

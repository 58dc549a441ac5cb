"""Why a plan does not capture (TDP_REPLAY_DEBUG=1 prints the exception)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ["TDP_REPLAY_DEBUG"] = "1"
import numpy as np

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200 import replay, workloads as wl

rng = np.random.default_rng(11)
n = 20_000
k = rng.integers(-10**12, 10**12, size=n)
v = rng.random(n)
cat = tq.Catalog()
cat.register("t", tq.table_from_columns(["k", "v"], [tq.plain(tq.Tensor(k)), tq.plain(tq.Tensor(v))]))
q = wl.compile_sql("SELECT k, SUM(v) FROM t GROUP BY k", cat, tq.UdfRegistry())
for _ in range(3):
    q.run(cat)
print("groupby:", [type(e).__name__ if not isinstance(e, str) else e for e in q._replays.values()])
tables = wl.q3_arrays(0.02, seed=7)
cat = wl.q3_catalog(tables)
plan = wl.Q3Plan(cat)
for _ in range(3):
    plan.run(cat)
print("q3:", [type(e).__name__ if not isinstance(e, str) else e for e in plan._pipeline._replays.values()])

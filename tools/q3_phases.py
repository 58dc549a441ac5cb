"""Host-side time per phase of the Q3-style pipeline (diagnostic only)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2211_02753_b200 import workloads as wl
from paper_2211_02753_b200.kernels import equi_join
from paper_2211_02753_b200.storage import Catalog, table_from_columns

tables = wl.q3_arrays(10.0, seed=7)
cat = wl.q3_catalog(tables)
plan = wl.Q3Plan(cat)
for _ in range(3):
    plan.run(cat)
torch.cuda.synchronize()
acc = {}
N = 20
for _ in range(N):
    t = [time.perf_counter()]
    c = plan.cust.run(cat); o = plan.orders.run(cat); li = plan.lineitem.run(cat)
    t.append(time.perf_counter())
    oc = equi_join(list(o.columns), list(c.columns), 1, 0, left_out=[0, 2, 3], right_out=[])
    t.append(time.perf_counter())
    j = equi_join(list(li.columns), oc, 0, 0, right_out=[1, 2])
    t.append(time.perf_counter())
    names = ["l_orderkey", "l_extendedprice", "l_discount", "o_orderdate", "o_shippriority"]
    work = Catalog()
    work.register("joined", table_from_columns(names, j))
    res = plan.tail.run(work)
    t.append(time.perf_counter())
    _ = res.columns[0].values.numpy()
    t.append(time.perf_counter())
    for k, (a, b) in enumerate(zip(t, t[1:])):
        acc[k] = acc.get(k, 0.0) + (b - a)
for k, name in enumerate(["3 filter queries", "join orders-customer", "join lineitem-orders",
                          "tail query (group/order/limit)", "result read"]):
    print(f"{name:32s} {acc[k] / N * 1e3:7.3f} ms (host, incl. waits at syncs)")

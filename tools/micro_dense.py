"""Microbenchmark of the dense-range join build on the Q3 orders table
(diagnostic): per-kernel device time by torch.profiler for variants of the
build (unfiltered / date filter / date + semi-join bitmap; with and without
the build-row index)."""
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200 import kernels as K, workloads as wl

tables = wl.q3_arrays(10.0, seed=7)
cat = wl.q3_catalog(tables)
o = cat.get("orders")
c = cat.get("customer")
li = cat.get("lineitem")
cust = K.filter_exact(list(c.columns), [(1, "=", "BUILDING")])
semi = K.equi_join(list(o.columns), cust, 1, 0, right_out=[])
date = K.filter_exact(list(o.columns), [(2, "<", 9204)])
probe = K.filter_exact(list(li.columns), [(1, ">", 9204)])
cases = {
    "unfiltered_rows": (list(o.columns), [1]),
    "unfiltered_norows": (list(o.columns), []),
    "date_rows": (date, [1]),
    "date_semi_rows": (K.equi_join(date, cust, 1, 0, right_out=[]), [1, 2]),
}
for name, (build, ro) in cases.items():
    for _ in range(2):
        K.equi_join(probe, build, 0, 0, left_out=[0], right_out=ro)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            K.equi_join(probe, build, 0, 0, left_out=[0], right_out=ro)
        torch.cuda.synchronize()
    agg = defaultdict(float)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            agg[e.name[:60]] += (e.device_time_total if hasattr(e, "device_time_total")
                                 else e.cuda_time_total) / 3
    print(f"== {name}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:6]:
        print(f"   {v:8.1f} us  {k}")

"""In-situ kernel-time breakdown of the Q3-style pipeline (torch.profiler CUDA
activity; diagnostic only -- no number here is a bench value)."""
import sys
import time
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2211_02753_b200 import workloads as wl

sf = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
tables = wl.q3_arrays(sf, seed=7)
cat = wl.q3_catalog(tables)
plan = wl.Q3Plan(cat)
for _ in range(3):
    plan.run(cat)
torch.cuda.synchronize()
N = 5
t0 = time.perf_counter()
for _ in range(N):
    plan.run(cat)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / N * 1e3
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(N):
        plan.run(cat)
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        a = agg[e.name[:90]]
        a[0] += 1
        a[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
tot = sum(v[1] for v in agg.values())
print(f"wall {wall:.3f} ms/run; device busy {tot / N / 1e3:.3f} ms/run")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{c // N:4d}x {t / N:9.1f} us/run {100 * t / tot:5.1f}%  {k}")
print("per-launch (last run):")
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
per_run = len(evs) // N
for e in evs[-per_run:]:
    t = e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    if t > 20:
        print(f"  {t:8.1f} us  {e.name[:80]}")

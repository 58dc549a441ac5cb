"""GPU idle gaps inside LLP train() iterations at 1e8 x 64 (diagnostic)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200.storage import tensor_type
from paper_2211_02753_b200.training import TrainConfig

n, d, bags = 100_000_000, 64, 1000
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(n, d, generator=g, device="cuda")
bag = torch.randint(0, bags, (n,), generator=g, device="cuda")
target = torch.rand(bags * 2, device="cuda", dtype=torch.float64) * 1e5
model = tq.Linear(d, 2, np.random.default_rng(0), name="lin")
bag_pe = tq.one_hot_pe(bag, bags)
reg = tq.UdfRegistry()
reg.register(tq.UdfEntry("llp", (("Bag", tensor_type(bags)), ("Pred", tensor_type(2))), 1,
                         lambda c: (bag_pe, tq.pe_encode(model(c.values))), model.parameters))
cat = tq.Catalog()
Xt = tq.Tensor(X)
cat.register_tensor(Xt, "T")
q = tq.compile_plan(tq.lower(tq.bind(tq.parse("SELECT Bag, Pred, COUNT(*) FROM llp(T) GROUP BY Bag, Pred"),
                                     cat, reg)), tq.CompileConfig(trainable=True), reg)
batches = [("T", Xt, tq.Tensor(target))]
tq.train(q, cat, batches, TrainConfig(iterations=3))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    tq.train(q, cat, batches, TrainConfig(iterations=3))
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda e: e.time_range.start)
span = (evs[-1].time_range.end - evs[0].time_range.start) / 3
busy = sum(e.time_range.end - e.time_range.start for e in evs) / 3
print(f"per iteration: span {span / 1e3:.3f} ms, busy {busy / 1e3:.3f} ms, kernels {len(evs) // 3}")
gaps = []
for a, b in zip(evs, evs[1:]):
    gap = b.time_range.start - a.time_range.end
    gaps.append((gap, a.name[:60], b.name[:60]))
for gap, a, b in sorted(gaps, reverse=True)[:12]:
    print(f"  gap {gap:8.1f} us  after {a}  before {b}")

import time
for iters in (5, 20, 40):
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    tq.train(q, cat, batches, TrainConfig(iterations=iters))
    t1.record()
    torch.cuda.synchronize()
    print(f"train({iters}): {t0.elapsed_time(t1) / iters:.3f} ms per iteration")

"""Kernel-time breakdown of one LLP trainable step (torch.profiler; diagnostic only)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200.storage import tensor_type
from paper_2211_02753_b200.training import AdamState, TrainConfig, train_step

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
d, bags = 64, 1000
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(n, d, generator=g, device="cuda")
bag = torch.randint(0, bags, (n,), generator=g, device="cuda")
target = torch.rand(bags * 2, device="cuda", dtype=torch.float64) * (n / bags / 2)
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
params = q.parameters()
cfg = TrainConfig(iterations=1, lr=0.01)
state = AdamState.for_params(params)
tgt = tq.Tensor(target)
for _ in range(3):
    train_step(q, cat, "T", Xt, tgt, params, cfg, state)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        train_step(q, cat, "T", Xt, tgt, params, cfg, state)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=20, max_name_column_width=70))

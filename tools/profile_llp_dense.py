"""Kernel breakdown of the dense-head (K=1000) LLP step at 1e7 rows
(torch.profiler; diagnostic only)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200.storage import tensor_type
from paper_2211_02753_b200.training import TrainConfig

torch.backends.cuda.matmul.allow_tf32 = False
n, d, k = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000, 64, 1000
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(n, d, generator=g, device="cuda")
target = torch.full((k,), n / k, dtype=torch.float64, device="cuda")
model = tq.Linear(d, k, np.random.default_rng(0), name="lin")
reg = tq.UdfRegistry()
reg.register(tq.UdfEntry("clf", (("Pred", tensor_type(k)),), 1,
                         lambda c: (tq.pe_encode(model(c.values)),), model.parameters))
cat = tq.Catalog()
Xt = tq.Tensor(X)
cat.register_tensor(Xt, "T")
q = tq.compile_plan(tq.lower(tq.bind(tq.parse("SELECT Pred, COUNT(*) FROM clf(T) GROUP BY Pred"),
                                     cat, reg)), tq.CompileConfig(trainable=True), reg)
from paper_2211_02753_b200 import autograd as AG
AG.WIDE_HEAD_BYTES = 0
tq.train(q, cat, [("T", Xt, tq.Tensor(target))], TrainConfig(iterations=1, lr=0.01))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    tq.train(q, cat, [("T", Xt, tq.Tensor(target))], TrainConfig(iterations=1, lr=0.01))
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15, max_name_column_width=80))

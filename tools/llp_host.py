"""Host time per LLP train() iteration at small n (GPU time ~0): where does
the step's non-kernel time go?  (diagnostic only)"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200.storage import tensor_type
from paper_2211_02753_b200.training import TrainConfig

n, d, bags = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, 64, 1000
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(n, d, generator=g, device="cuda")
bag = torch.randint(0, bags, (n,), generator=g, device="cuda")
target = torch.rand(bags * 2, device="cuda", dtype=torch.float64)
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
tq.train(q, cat, batches, TrainConfig(iterations=5))
torch.cuda.synchronize()
t0 = time.perf_counter()
tq.train(q, cat, batches, TrainConfig(iterations=50))
torch.cuda.synchronize()
print(f"n={n}: {(time.perf_counter() - t0) / 50 * 1e3:.3f} ms per iteration (wall)")
pr = cProfile.Profile()
pr.enable()
tq.train(q, cat, batches, TrainConfig(iterations=20))
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(20)

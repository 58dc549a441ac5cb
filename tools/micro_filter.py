"""Micro-benchmark: materialising filter (tdp_filter_select) on one int64
column, CUDA-event timed (diagnostic; not a bench value)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200.kernels import filter_exact


def run(col, lit, label):
    c = tq.plain(tq.Tensor(col))
    for _ in range(3):
        out = filter_exact([c], [(0, "<", lit)])
        out[0].values._lazy.sel.indices()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 20
    e0.record()
    for _ in range(R):
        out = filter_exact([c], [(0, "<", lit)])
        idx = out[0].values._lazy.sel.indices()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    n = col.numel()
    print(f"{label} n={n}: {ms:.3f} ms  ({n * 8 / ms / 1e6:.0f} GB/s of predicate column), "
          f"selected {idx.numel()}")


for n in (1_500_000, 15_000_000, 60_000_000):
    run(torch.randint(0, 10000, (n,), dtype=torch.int64, device="cuda"), 5000, "random")
rng = np.random.default_rng(7)
od = rng.integers(8035, 10440 + 1, size=15_000_000, dtype=np.int64)
run(tq.Tensor(od).data, 9204, "q3-orders")

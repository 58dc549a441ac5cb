"""One partitioned bitmap group-by (2^22 + 5 rows) for compute-sanitizer
(memcheck / racecheck / synccheck of part_*_kernel).  Run on the GPU box:
compute-sanitizer --tool memcheck python tools/sanitize_partition.py"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200.kernels import groupby_exact

rng = np.random.default_rng(5)
n = (1 << 22) + 5
key = rng.integers(0, 3_000_000, size=n).astype(np.int64)
fv = rng.normal(size=n)
iv = rng.integers(-1000, 1000, size=n)
kv, aggs = groupby_exact([tq.plain(tq.Tensor(key))],
                         [("sum", tq.Tensor(fv)), ("sum", tq.Tensor(iv)), ("count", None)])
torch.cuda.synchronize()
cnt = aggs[2].cpu().numpy()
assert int(cnt.sum()) == n and len(cnt) == len(np.unique(key))
print("ok", len(cnt))

import sys
sys.path.insert(0, '/root/repo')
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2211_02753_b200 as tq
from paper_2211_02753_b200 import kernels as K
n = 60_000_000
g = torch.Generator(device="cuda").manual_seed(0)
f64 = torch.rand(n, generator=g, device="cuda", dtype=torch.float64)
keys = torch.randint(0, 1_000_000, (n,), generator=g, device="cuda") * 1_000_003 + 7
kb = torch.randint(0, 5_000_000, (n,), generator=g, device="cuda")
ops = {
 "hash": lambda: K.groupby_exact([tq.plain(tq.Tensor(keys))], [("sum", tq.Tensor(f64)), ("count", None)]),
 "hash_count_only": lambda: K.groupby_exact([tq.plain(tq.Tensor(keys))], [("count", None)]),
 "bitmap": lambda: K.groupby_exact([tq.plain(tq.Tensor(kb))], [("sum", tq.Tensor(f64)), ("count", None)]),
 "bitmap_count_only": lambda: K.groupby_exact([tq.plain(tq.Tensor(kb))], [("count", None)]),
 "bitmap_int_sum": lambda: K.groupby_exact([tq.plain(tq.Tensor(kb))], [("sum", tq.Tensor(keys)), ("count", None)]),
 "topk": lambda: K.topk_order(tq.plain(tq.Tensor(f64)), 10, True),
}
for name, fn in ops.items():
    fn(); fn(); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn(); torch.cuda.synchronize()
    print("=====", name)
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=8, max_name_column_width=70))

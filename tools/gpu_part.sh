timeout 900 python -m pytest tests/test_gpu_queries.py -q -x -k "partitioned or bitmap or float_group_sums" > gpurun_out/pt_part.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_part.log; grep -E "^E  " gpurun_out/pt_part.log | head -20
for m in 1 0; do TDP_GROUPBY_PARTITION=$m timeout 600 python tools/kernel_zoo.py 2>&1 | grep -i "groupby"; done
timeout 300 python - <<'PY'
import torch, paper_2211_02753_b200 as tq
from paper_2211_02753_b200 import kernels as K
from torch.profiler import profile, ProfilerActivity
n=60_000_000
g=torch.Generator(device="cuda").manual_seed(0)
kb=torch.randint(0,5_000_000,(n,),generator=g,device="cuda"); f=torch.rand(n,generator=g,device="cuda",dtype=torch.float64)
c=tq.plain(tq.Tensor(kb))
fn=lambda: K.groupby_exact([c],[("sum",tq.Tensor(f)),("count",None)])
for _ in range(2): fn()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    fn(); torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=12, max_name_column_width=60))
PY

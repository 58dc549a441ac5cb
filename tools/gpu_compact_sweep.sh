# Compact-storage Q1/Q6 kernel under ring shapes (measurement helper).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_queries.py -x -q > gpurun_out/pytest_compact.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_compact.log
for cfg in "TDP_VEC_PU=8" "TDP_VEC_PU=4" "TDP_VEC_PU=8 TDP_NARROW_CTAS=3"; do
  env $cfg timeout 600 python bench.py --encoding compact --steps 200 --warmup 5 --no-cpu-baseline --no-parity > gpurun_out/sweep.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/sweep.json').read().strip().splitlines()[-1])
print('$cfg', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['companion_q6']['kernel_ms'])"
done

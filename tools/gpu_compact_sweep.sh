# Compact-storage Q1/Q6 kernel under codegen variants (measurement helper).
mkdir -p gpurun_out
for cfg in "TDP_VEC_PU=8" "TDP_VEC_PU=4"; do
  env $cfg timeout 600 python bench.py --encoding compact --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/sweep.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/sweep.json').read().strip().splitlines()[-1])
print('$cfg', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['companion_q6']['kernel_ms'], d['parity']['status'], d['parity'].get('max_rel_err'))"
done

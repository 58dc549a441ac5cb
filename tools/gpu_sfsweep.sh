mkdir -p gpurun_out
for sf in 1 3 10 30; do timeout 900 python bench.py --sf $sf --steps 200 --e2e-steps 2 --no-cpu-baseline --no-companion > gpurun_out/sweep_q1_sf$sf.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/sweep_q1_sf$sf.json')); r=d['roofline']
print('Q1 SF$sf rows %d step %.4f ms  kernel %.4f ms  %.0f GB/s  frac %.3f  value %.3g rows/s  e2e %.3g' % (d['config']['rows'], d['ms_per_step'], r['kernel_ms'], r['achieved'], r['frac'], d['value'], d['e2e']['value']))"; done

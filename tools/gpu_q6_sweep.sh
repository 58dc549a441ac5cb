# Q6 SF1 / SF10 ring-shape sweep (measurement knobs of pipeline.cu)
mkdir -p gpurun_out
run() { local tag=$1; shift; for sf in 1 10; do env "$@" timeout 300 python bench.py --query q6 --sf $sf --steps 200 --warmup 5 --no-companion --no-cpu-baseline --no-parity --e2e-steps 1 > gpurun_out/q6.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/q6.json'));r=d['roofline'];print('$tag sf$sf step',round(d['ms_per_step']*1e3,1),'us kernel',round(r['kernel_ms']*1e3,1),'us frac',round(r['frac'],3))"; done; }
run default X=1
run onecta TDP_TWO_CTA_ROW_BYTES=0
run budget220 TDP_TWO_CTA_ROW_BYTES=0 TDP_RING_BUDGET_KB=220
run default2 X=1

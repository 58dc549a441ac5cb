mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for q in "--query q1" "--query q1 --encoding compact" "--query q6 --sf 1" "--query q3"; do
timeout 600 python bench.py $q --steps 100 --warmup 5 --no-companion --no-cpu-baseline --e2e-steps 1 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "import json;d=json.load(open('gpurun_out/b.json'));r=d['roofline'];print('$q step',round(d['ms_per_step']*1e3,1),'us kernel',round(r['kernel_ms']*1e3,1), d['parity']['status'])"
done

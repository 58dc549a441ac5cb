mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "runs or bitmap or groupby or q3 or golden" > gpurun_out/pt_runs.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pt_runs.log | grep -v "^$" | tail -25
timeout 600 python bench.py --query q3 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/q3.json 2>gpurun_out/q3.err; echo "q3 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/q3.json'));r=d['roofline'];print('step',round(d['ms_per_step'],4),'eager',round(d['eager_ms_per_step'],4),'probe',round(r['kernel_ms'],4),r['frac'],d['parity'],'launches/step',d['gpu_launches']/d['steps'])"

# full GPU suite + Q3 bench line + Q3 launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --query q3 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/q3.json 2>gpurun_out/q3.err; echo "q3 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/q3.json'));r=d['roofline'];print('step',round(d['ms_per_step'],4),'eager',round(d['eager_ms_per_step'],4),'probe',round(r['kernel_ms'],4),r['frac'],d['parity']['status'],'launches/step',d['gpu_launches']/d['steps'])"
TDP_REPLAY=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_q3.csv python tools/profile_q3.py 10 > /dev/null 2>&1; echo "ncu list rc=$?"

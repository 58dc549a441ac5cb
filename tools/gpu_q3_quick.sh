mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "join or q3 or semi or dense" > gpurun_out/pt_join.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt_join.log
for i in 1 2; do
timeout 600 python bench.py --query q3 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/q3.json 2>gpurun_out/q3.err
python -c "import json;d=json.load(open('gpurun_out/q3.json'));r=d['roofline'];print('step',round(d['ms_per_step'],4),'probe',round(r['kernel_ms'],4),r['frac'],d['parity']['status'],'launches/step',d['gpu_launches']/d['steps'])"
done
TDP_REPLAY=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:dense_build --csv --log-file gpurun_out/build.csv python tools/profile_q3.py 10 > /dev/null 2>&1
python tools/launches.py gpurun_out/build.csv | head -3

mkdir -p gpurun_out/san
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do
timeout 600 python bench.py --query q3 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/q3.json 2>gpurun_out/q3.err
python -c "import json;d=json.load(open('gpurun_out/q3.json'));r=d['roofline'];print('step',round(d['ms_per_step'],4),'eager',round(d['eager_ms_per_step'],4),'probe',round(r['kernel_ms'],4),r['frac'],d['parity']['status'],'launches/step',d['gpu_launches']/d['steps'])"
done
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_csv.py tests/test_gpu_join.py -x -q -p no:cacheprovider -k "device_csv_equals or sorted_join_large or adversarial" > gpurun_out/san/racecheck_r02_csv_join.txt 2>&1; echo "racecheck csv/join rc=$?"; tail -2 gpurun_out/san/racecheck_r02_csv_join.txt
timeout 1200 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_join.py tests/test_gpu_queries.py -x -q -p no:cacheprovider -k "join or q3 or runs" > gpurun_out/san/memcheck_r02_join_fused_emit.txt 2>&1; echo "memcheck join rc=$?"; tail -2 gpurun_out/san/memcheck_r02_join_fused_emit.txt

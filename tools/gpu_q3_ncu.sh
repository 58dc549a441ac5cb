# Q3: bench line, join GPU tests, ncu --set full of the orders build and the lineitem probe
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "join or q3 or semi" > gpurun_out/pt_join.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_join.log
timeout 600 python bench.py --query q3 --steps 50 --warmup 5 > gpurun_out/q3.json 2>gpurun_out/q3.err; echo "q3 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/q3.json'));r=d['roofline'];print('step',round(d['ms_per_step'],4),'eager',round(d['eager_ms_per_step'],4),'probe',round(r['kernel_ms'],4),r['frac'],d['parity']['status'])"
TDP_REPLAY=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_build_kernel --launch-skip 1 -c 1 -o gpurun_out/q3_build python tools/profile_q3.py 10 > /dev/null 2>&1; echo "ncu build rc=$?"
TDP_REPLAY=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_count_kernel --launch-skip 2 -c 1 -o gpurun_out/q3_probe python tools/profile_q3.py 10 > /dev/null 2>&1; echo "ncu probe rc=$?"
TDP_REPLAY=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_q3.csv python tools/profile_q3.py 10 > /dev/null 2>&1; echo "ncu list rc=$?"

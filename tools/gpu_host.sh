mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_replay.py tests/test_gpu_nccl.py -x -q > gpurun_out/pt_replay.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_replay.log
timeout 300 python tools/profile_replay_host.py q6 1 > gpurun_out/host_q6.txt 2>&1; echo "prof rc=$?"; head -1 gpurun_out/host_q6.txt
timeout 600 python bench.py --query q6 --sf 1 --steps 200 --warmup 5 --no-companion --no-cpu-baseline > gpurun_out/q6sf1.json 2>gpurun_out/q6sf1.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/q6sf1.json'));r=d['roofline'];print('step',round(d['ms_per_step'],4),'kernel',round(r['kernel_ms'],4),r['frac'],d['parity']['status'])"

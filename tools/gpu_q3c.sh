mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --query q3 > gpurun_out/bench_q3.json 2> gpurun_out/bench_q3.err; echo "q3 rc=$?"; cut -c1-250 gpurun_out/bench_q3.json; tail -3 gpurun_out/bench_q3.err
TDP_REPLAY=0 timeout 300 python tools/profile_host.py q1 2>&1 | head -2
timeout 300 python tools/profile_host.py q1 2>&1 | head -2

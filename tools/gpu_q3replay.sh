mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_replay.py tests/test_gpu_queries.py -x -q 2>&1 | tail -5
timeout 300 python bench.py --query q3 --steps 20 --warmup 3 > gpurun_out/bench_q3.json 2> gpurun_out/bench_q3.err; cat gpurun_out/bench_q3.json | cut -c1-400; tail -3 gpurun_out/bench_q3.err
timeout 300 python tools/profile_q3.py 10 2>/dev/null | head -4

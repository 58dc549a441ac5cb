mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/profile_q3.py 10 > gpurun_out/q3prof.txt 2>&1; head -30 gpurun_out/q3prof.txt
timeout 600 python bench.py --query q3 > gpurun_out/bench_q3.json 2> gpurun_out/bench_q3.err; echo "q3 rc=$?"; cut -c1-300 gpurun_out/bench_q3.json; tail -3 gpurun_out/bench_q3.err

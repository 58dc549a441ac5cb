mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_soft_linear.py tests/test_gpu_llp.py tests/test_gpu_soft.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --query llp > gpurun_out/bench_llp.json 2> gpurun_out/bench_llp.err; echo "llp rc=$?"; cat gpurun_out/bench_llp.json | cut -c1-400
timeout 300 python tools/profile_llp.py > gpurun_out/llpprof.txt 2>&1; grep -E "soft_linear|wgrad" gpurun_out/llpprof.txt | cut -c1-70,150-240

mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_llp.py tests/test_gpu_image_query.py tests/test_gpu_golden.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --query llp > gpurun_out/bench_llp.json 2> gpurun_out/bench_llp.err; echo "llp rc=$?"; cat gpurun_out/bench_llp.json | cut -c1-300; tail -3 gpurun_out/bench_llp.err

mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_image_query.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --query image --image-rows 1000000 > gpurun_out/bench_image_1m.json 2> gpurun_out/bench_image_1m.err; echo "rc=$?"; cat gpurun_out/bench_image_1m.json; tail -3 gpurun_out/bench_image_1m.err
timeout 900 python bench.py --query image > gpurun_out/bench_image.json 2> gpurun_out/bench_image.err; echo "rc=$?"; cat gpurun_out/bench_image.json; tail -3 gpurun_out/bench_image.err

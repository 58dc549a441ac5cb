mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1 TDP_REPLAY=0
timeout 1700 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_queries.py tests/test_gpu_compact.py tests/test_gpu_golden.py tests/test_gpu_soft.py tests/test_gpu_soft_linear.py tests/test_gpu_llp.py -x -q -k "not 3_000_000 and not 1_000_003 and not replay" > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"; grep -v "Host Frame" gpurun_out/memcheck.log | tail -30

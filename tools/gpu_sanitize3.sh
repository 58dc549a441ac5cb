mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1 TDP_REPLAY=0
timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 --error-exitcode 9 python -m pytest tests/test_gpu_queries.py -x -q -k "hash_groupby or q3 or join" > gpurun_out/memcheck3.log 2>&1; echo "memcheck rc=$?"; grep -v "Host Frame" gpurun_out/memcheck3.log | tail -3
timeout 1200 compute-sanitizer --tool racecheck --print-limit 10 --error-exitcode 9 python -m pytest tests/test_gpu_queries.py -x -q -k "hash_groupby_bitmap" > gpurun_out/racecheck3.log 2>&1; echo "racecheck rc=$?"; grep -v "Host Frame" gpurun_out/racecheck3.log | tail -3

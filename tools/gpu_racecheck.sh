mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1 TDP_REPLAY=0
timeout 1700 compute-sanitizer --tool racecheck --print-limit 10 --error-exitcode 9 python -m pytest tests/test_gpu_queries.py tests/test_gpu_soft_linear.py -x -q -k "topk or hash_groupby or filtered_build or q1_matches or q6_matches or soft_linear" > gpurun_out/racecheck.log 2>&1; echo "racecheck rc=$?"; grep -v "Host Frame" gpurun_out/racecheck.log | tail -20
timeout 900 compute-sanitizer --tool synccheck --print-limit 10 --error-exitcode 9 python -m pytest tests/test_gpu_queries.py -x -q -k "topk or q1_matches" > gpurun_out/synccheck.log 2>&1; echo "synccheck rc=$?"; grep -v "Host Frame" gpurun_out/synccheck.log | tail -8

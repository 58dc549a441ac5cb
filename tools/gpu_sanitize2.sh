mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1 TDP_REPLAY=0
timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 --error-exitcode 9 python -m pytest tests/test_gpu_queries.py -x -q -k "topk or order or limit or q3 or join or q1_matches" > gpurun_out/memcheck2.log 2>&1; echo "memcheck rc=$?"; grep -v "Host Frame" gpurun_out/memcheck2.log | tail -5
timeout 1200 compute-sanitizer --tool racecheck --print-limit 10 --error-exitcode 9 python -m pytest tests/test_gpu_queries.py -x -q -k "topk or order or q1_matches" > gpurun_out/racecheck2.log 2>&1; echo "racecheck rc=$?"; grep -v "Host Frame" gpurun_out/racecheck2.log | tail -5
timeout 900 compute-sanitizer --tool synccheck --print-limit 10 --error-exitcode 9 python -m pytest tests/test_gpu_queries.py -x -q -k "topk or q1_matches" > gpurun_out/synccheck2.log 2>&1; echo "synccheck rc=$?"; grep -v "Host Frame" gpurun_out/synccheck2.log | tail -4

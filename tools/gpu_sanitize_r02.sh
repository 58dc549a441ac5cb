# Round-2 compute-sanitizer runs over the kernels added this round (device CSV,
# sorted join, dense join build + probe with the L2 run-ahead, exact packed
# scan, one-pass LLP, soft sort, device dict_encode, sorted-runs group-by,
# top-k with fused key images, AVG in the emit kernels).  Output: gpurun_out/san/.
O=gpurun_out/san; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_gpu_csv.py tests/test_gpu_join.py tests/test_gpu_compact.py tests/test_gpu_llp_onepass.py tests/test_gpu_softsort.py tests/test_gpu_integration.py"
timeout 1500 $CS --tool memcheck --error-exitcode 9 python -m pytest $T -x -q -p no:cacheprovider > $O/memcheck_r02.txt 2>&1; echo "memcheck rc=$?"; tail -3 $O/memcheck_r02.txt
timeout 1200 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_queries.py -x -q -p no:cacheprovider -k "runs or bitmap or topk or limit or order or hash" > $O/memcheck_r02_groupby_topk.txt 2>&1; echo "memcheck2 rc=$?"; tail -3 $O/memcheck_r02_groupby_topk.txt
timeout 1200 $CS --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_csv.py tests/test_gpu_compact.py tests/test_gpu_join.py -x -q -p no:cacheprovider -k "device_csv_equals or decimal_sums or sorted_join_large or adversarial" > $O/racecheck_r02.txt 2>&1; echo "racecheck rc=$?"; tail -3 $O/racecheck_r02.txt
timeout 1200 $CS --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_queries.py -x -q -p no:cacheprovider -k "runs or topk or limit" > $O/racecheck_r02_runs_topk.txt 2>&1; echo "racecheck2 rc=$?"; tail -3 $O/racecheck_r02_runs_topk.txt
timeout 900 $CS --tool synccheck python -m pytest tests/test_gpu_compact.py tests/test_gpu_llp_onepass.py -x -q -p no:cacheprovider > $O/synccheck_r02.txt 2>&1; echo "synccheck rc=$?"; tail -3 $O/synccheck_r02.txt

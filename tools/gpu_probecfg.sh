mkdir -p gpurun_out
for c in 0 1 2 3; do echo "== cfg $c"
TDP_JOIN_PROBE_CFG=$c TDP_REPLAY=0 timeout 300 python tools/profile_q3.py 10 2>/dev/null | grep -E "wall|join_count"
done
TDP_JOIN_PROBE_CFG=1 timeout 300 python -m pytest tests/test_gpu_queries.py -x -q -k "join or q3" 2>&1 | tail -1

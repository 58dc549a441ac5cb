mkdir -p gpurun_out
for v in 0 1 2; do echo "== variant $v"
TDP_JOIN_PREFETCH=0 TDP_JOIN_VARIANT=$v timeout 300 python tools/profile_q3.py 10 2>/dev/null | grep -E "wall|join_count"
done

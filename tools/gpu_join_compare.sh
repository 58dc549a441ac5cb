# Q3 SF10 with the default joins (dense-range / hash) vs the sort/searchsorted
# join (TDP_JOIN_ALGO=sort): bench lines + ncu launch lists (per-kernel time
# and DRAM bytes, cold-cache, serialised).  Output: gpurun_out/join_cmp/.
O=gpurun_out/join_cmp; mkdir -p $O
for algo in auto sort; do
  TDP_JOIN_ALGO=$algo timeout 600 python bench.py --query q3 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_q3_$algo.json 2> $O/bench_q3_$algo.err; echo "bench $algo rc=$?"
  TDP_JOIN_ALGO=$algo TDP_REPLAY=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_q3_$algo.csv python tools/profile_q3.py 10 > /dev/null 2>&1; echo "ncu $algo rc=$?"
done

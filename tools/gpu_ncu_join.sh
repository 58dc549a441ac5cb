mkdir -p gpurun_out
TDP_JOIN_PREFETCH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_count -s 4 -c 2 \
   -o gpurun_out/q3_join2 -f python tools/profile_q3.py 10 > gpurun_out/ncu_q3.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/ncu_q3.log

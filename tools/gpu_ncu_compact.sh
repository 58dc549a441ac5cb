mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tdp_scan_agg -s 5 -c 1 \
   -o gpurun_out/q1c_now -f python bench.py --query q1 --encoding compact --steps 3 --warmup 3 --no-cpu-baseline --no-companion > gpurun_out/ncu_q1c.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/ncu_q1c.log

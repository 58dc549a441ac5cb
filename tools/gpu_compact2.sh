mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_compact.py -x -q 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tdp_scan_agg -s 2 -c 1 -o gpurun_out/q1c_prof -f python bench.py --query q1 --encoding compact --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_q1c.log 2>&1; tail -2 gpurun_out/ncu_q1c.log

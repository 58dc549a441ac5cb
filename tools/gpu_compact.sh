mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_compact.py tests/test_gpu_queries.py tests/test_gpu_golden.py -x -q 2>&1 | tail -15
for q in q1 q6; do timeout 600 python bench.py --query $q --encoding compact --steps 300 > gpurun_out/bench_${q}_compact.json 2> gpurun_out/bench_${q}_compact.err; echo "$q rc=$?"; cut -c1-300 gpurun_out/bench_${q}_compact.json; grep -o '"e2e.\{1,120\}\|"roofline.\{1,260\}' gpurun_out/bench_${q}_compact.json; tail -3 gpurun_out/bench_${q}_compact.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tdp_scan_agg -s 8 -c 1 -o gpurun_out/q1c_prof -f python bench.py --query q1 --encoding compact --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_q1c.log 2>&1; tail -2 gpurun_out/ncu_q1c.log

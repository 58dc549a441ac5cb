mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_compact.py tests/test_gpu_queries.py -x -q 2>&1 | tail -3
for q in q1 q6; do timeout 600 python bench.py --query $q --encoding compact --steps 300 --no-cpu-baseline > gpurun_out/bench_${q}_compact.json 2> gpurun_out/bench_${q}_compact.err; echo "$q rc=$?"; grep -o '"ms_per_step.\{1,30\}\|"e2e.\{1,60\}\|"achieved.\{1,90\}\|kernel_ms.\{1,30\}' gpurun_out/bench_${q}_compact.json; tail -3 gpurun_out/bench_${q}_compact.err; done
timeout 600 python bench.py --query q1 --steps 200 --no-cpu-baseline > gpurun_out/bench_q1.json 2> gpurun_out/bench_q1.err; grep -o '"ms_per_step.\{1,30\}\|"achieved.\{1,90\}\|kernel_ms.\{1,30\}' gpurun_out/bench_q1.json

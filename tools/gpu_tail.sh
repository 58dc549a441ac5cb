mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_q1.json 2> gpurun_out/bench_q1.err; echo "q1 rc=$?"; grep -o '"value.\{1,30\}\|"ms_per_step.\{1,30\}\|"e2e.\{1,60\}\|kernel_ms.\{1,30\}\|"companion_q6.\{1,300\}\|"parity.\{1,30\}' gpurun_out/bench_q1.json; tail -3 gpurun_out/bench_q1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/q1_launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-companion > gpurun_out/q1_ncu_bench.log 2>&1; echo "ncu rc=$?"

# Full bench lines for profiles/ (headline Q1 with cpu_baseline + parity, Q6, compact variants, reference arm)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python bench.py > gpurun_out/bench_q1.json 2> gpurun_out/bench_q1.err; echo "q1 rc=$?"; cut -c1-200 gpurun_out/bench_q1.json
timeout 600 python bench.py --query q6 > gpurun_out/bench_q6.json 2> gpurun_out/bench_q6.err; echo "q6 rc=$?"
timeout 600 python bench.py --encoding compact > gpurun_out/bench_q1_compact.json 2> gpurun_out/bench_q1_compact.err; echo "q1c rc=$?"
timeout 600 python bench.py --query q6 --encoding compact > gpurun_out/bench_q6_compact.json 2> gpurun_out/bench_q6_compact.err; echo "q6c rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref_q1.json 2> gpurun_out/ref_q1.err; echo "ref rc=$?"; cut -c1-200 gpurun_out/ref_q1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/q1_launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/q1_ncu_bench.log 2>&1; echo "ncu rc=$?"

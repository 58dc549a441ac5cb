# Full bench lines for profiles/ (headline Q1 with cpu_baseline + parity, Q6, compact variants,
# Q3, LLP, reference arm) and the fused-scan launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_q1.json 2> gpurun_out/bench_q1.err; echo "q1 rc=$?"
timeout 600 python bench.py --query q6 > gpurun_out/bench_q6.json 2> gpurun_out/bench_q6.err; echo "q6 rc=$?"
timeout 600 python bench.py --encoding compact > gpurun_out/bench_q1_compact.json 2> gpurun_out/bench_q1_compact.err; echo "q1c rc=$?"
timeout 600 python bench.py --query q6 --encoding compact > gpurun_out/bench_q6_compact.json 2> gpurun_out/bench_q6_compact.err; echo "q6c rc=$?"
timeout 600 python bench.py --query q3 > gpurun_out/bench_q3.json 2> gpurun_out/bench_q3.err; echo "q3 rc=$?"
timeout 600 python bench.py --query llp > gpurun_out/bench_llp.json 2> gpurun_out/bench_llp.err; echo "llp rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref_q1.json 2> gpurun_out/ref_q1.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/q1_launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-companion > gpurun_out/q1_ncu_bench.log 2>&1; echo "ncu rc=$?"
for f in bench_q1 bench_q6 bench_q1_compact bench_q6_compact bench_q3 bench_llp ref_q1; do echo "$f: $(cut -c1-160 gpurun_out/$f.json)"; done

# Round-2 closing evidence: GPU suite, smoke, every bench line, operator zoo,
# Q1 launch list.  Run from the repo root on the box.
O=gpurun_out/r02c; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
b() { local name=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo "$name rc=$?"; }
b q1_sf10 --steps 200 --warmup 5
b q1_default
b q6_sf10 --query q6 --steps 200 --warmup 5
b q6_sf1 --query q6 --sf 1 --steps 200 --warmup 5 --no-companion
b q1_sf10_compact --encoding compact --steps 200 --warmup 5
b q3_sf10 --query q3 --steps 50 --warmup 5
b llp_onepass --query llp --steps 10 --warmup 4
b llp_dense_1000 --query llp-dense --steps 3 --warmup 3
b reference_arm --impl reference --steps 3 --warmup 1
b image_1e7 --query image --steps 2 --warmup 1 --no-cpu-baseline
timeout 600 python tools/kernel_zoo.py > $O/kernel_zoo_6e7.jsonl 2> $O/kernel_zoo.err; echo "zoo rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_q1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1 > /dev/null 2>&1; echo "ncu q1 rc=$?"
ls $O

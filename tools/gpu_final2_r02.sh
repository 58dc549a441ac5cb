# After the partitioned group-by: full GPU suite, smoke, operator zoo, Q3 line.
O=gpurun_out/r02d; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python tools/kernel_zoo.py > $O/kernel_zoo_6e7.jsonl 2> $O/kernel_zoo.err; echo "zoo rc=$?"
timeout 900 python bench.py --query q3 --steps 50 --warmup 5 > $O/bench_q3_sf10.json 2> $O/bench_q3_sf10.err; echo "q3 rc=$?"

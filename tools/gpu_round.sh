# One GPU-box session: tests, smoke, host profile, bench lines for every config.
# usage (from the repo root on the box): bash tools/gpu_round.sh [queries...]
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 300 python tools/profile_host.py q1 > gpurun_out/host_q1.txt 2>&1; head -40 gpurun_out/host_q1.txt
QS=${@:-q1 q6 q3 llp}
for q in $QS; do timeout 600 python bench.py --query $q > gpurun_out/bench_$q.json 2> gpurun_out/bench_$q.err; echo "$q rc=$?"; tail -c 2500 gpurun_out/bench_$q.json; echo; done

# Generic GPU-box session: pytest -m gpu (optional filter) then bench lines.
# usage: bash tools/gpu_run.sh "<pytest -k expr or 'all' or 'none'>" "<bench args>;<bench args>;..."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
K="$1"
if [ "$K" != "none" ]; then
  if [ "$K" = "all" ]; then timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
  else timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1; fi
  echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
fi
IFS=';' read -ra BENCHES <<< "$2"
i=0
for b in "${BENCHES[@]}"; do
  [ -z "$b" ] && continue
  i=$((i+1))
  timeout 900 python bench.py $b > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err
  echo "bench [$b] rc=$?"; tail -c 3000 gpurun_out/bench_$i.json; tail -3 gpurun_out/bench_$i.err; echo
done

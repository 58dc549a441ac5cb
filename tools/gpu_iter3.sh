mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "runs or rank_mode or dense_join" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
timeout 300 python tools/trace_plan.py q1 1 > gpurun_out/trace_q1.txt 2>&1; echo "trace rc=$?"
timeout 300 python tools/trace_plan.py q6 1 > gpurun_out/trace_q6.txt 2>&1; echo "trace rc=$?"

mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
for q in q1 q6; do for e in wide compact; do timeout 600 python bench.py --query $q --encoding $e --steps 300 --no-cpu-baseline > gpurun_out/bench_${q}_${e}.json 2> gpurun_out/bench_${q}_${e}.err; echo "$q $e rc=$?"; grep -o '"ms_per_step.\{1,30\}\|"e2e.\{1,60\}\|"achieved.\{1,90\}\|kernel_ms.\{1,30\}\|gpu_launches.\{1,10\}' gpurun_out/bench_${q}_${e}.json; tail -3 gpurun_out/bench_${q}_${e}.err; done; done
timeout 300 python tools/profile_host.py q1 > gpurun_out/host_q1.txt 2>&1; head -3 gpurun_out/host_q1.txt

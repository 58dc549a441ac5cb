mkdir -p gpurun_out
nproc; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"; free -g | head -2
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref_q1.json 2> gpurun_out/ref_q1.err; echo "ref rc=$?"; cat gpurun_out/ref_q1.json; tail -3 gpurun_out/ref_q1.err
timeout 300 python tools/profile_llp.py > gpurun_out/llpprof.txt 2>&1; head -40 gpurun_out/llpprof.txt

mkdir -p gpurun_out
timeout 300 python tools/profile_q3.py 10 > gpurun_out/q3prof.txt 2>&1; cat gpurun_out/q3prof.txt | head -80

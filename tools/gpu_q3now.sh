mkdir -p gpurun_out
timeout 300 python tools/profile_q3.py 10 > gpurun_out/q3prof.txt 2>&1; head -45 gpurun_out/q3prof.txt
timeout 200 python tools/q3_phases.py > gpurun_out/q3phases.txt 2>&1; cat gpurun_out/q3phases.txt

mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:soft_linear_count -s 6 -c 2 \
   -o gpurun_out/llp_prof -f python tools/profile_llp.py 20000000 > gpurun_out/ncu_llp.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/ncu_llp.log

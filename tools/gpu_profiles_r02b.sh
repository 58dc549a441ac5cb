# Round-2 evidence refresh: GPU tests, every bench line, ncu launch lists and
# one --set full capture per dominant kernel.  Run from the repo root on the box.
O=gpurun_out/r02b; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
b() { local name=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo "$name rc=$?"; }
b q1_sf10 --steps 200 --warmup 5
b q6_sf10 --query q6 --steps 200 --warmup 5
b q6_sf1 --query q6 --sf 1 --steps 200 --warmup 5 --no-companion
b q1_sf10_compact --encoding compact --steps 200 --warmup 5
b q3_sf10 --query q3 --steps 50 --warmup 5
b llp --query llp --steps 10 --warmup 3
b reference_arm --impl reference --steps 3 --warmup 1
b image --query image --steps 2 --warmup 1 --no-cpu-baseline
TDP_FORCE_DIST=1 TDP_FORCE_COLLECTIVES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 200 --warmup 5 --no-cpu-baseline > $O/bench_q1_sf10_nccl_world1.json 2> $O/bench_q1_sf10_nccl_world1.err; echo "nccl rc=$?"
# launch lists (cold-cache, serialised: shares of the step)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_q1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1 > /dev/null 2>&1; echo "ncu q1 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_q1_compact.csv python bench.py --encoding compact --steps 2 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1 > /dev/null 2>&1; echo "ncu q1c rc=$?"
TDP_REPLAY=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_q3.csv python tools/profile_q3.py 10 > /dev/null 2>&1; echo "ncu q3 rc=$?"
# --set full of the dominant kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tdp_scan_agg --launch-skip 4 -c 1 -o $O/q1_scan python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-companion --e2e-steps 1 > /dev/null 2>&1; echo "ncu full q1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tdp_scan_agg --launch-skip 4 -c 1 -o $O/q1c_scan python bench.py --encoding compact --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-companion --e2e-steps 1 > /dev/null 2>&1; echo "ncu full q1c rc=$?"
TDP_REPLAY=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_count_kernel -c 1 --launch-skip 2 -o $O/q3_probe python tools/profile_q3.py 10 > /dev/null 2>&1; echo "ncu full q3 rc=$?"
ls $O
TDP_REPLAY=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_build_kernel -c 1 --launch-skip 1 -o $O/q3_build python tools/profile_q3.py 10 > /dev/null 2>&1; echo "ncu full q3 build rc=$?"
ls $O

# Round-2 evidence: bench lines, NCCL one-rank sharded line, SASS of the NVRTC scan kernel,
# ncu launch lists and DRAM traffic of the dominant kernels.  Run from the repo root on the box.
mkdir -p gpurun_out/r02
O=gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python bench.py --steps 200 --warmup 5 > $O/bench_q1_sf10.json 2> $O/bench_q1_sf10.err; echo "q1 rc=$?"
timeout 600 python bench.py --query q6 --sf 1 --steps 200 --warmup 5 --no-companion > $O/bench_q6_sf1.json 2> $O/bench_q6_sf1.err; echo "q6sf1 rc=$?"
timeout 600 python bench.py --query q6 --steps 200 --warmup 5 > $O/bench_q6_sf10.json 2> $O/bench_q6_sf10.err; echo "q6 rc=$?"
timeout 600 python bench.py --encoding compact --steps 200 --warmup 5 > $O/bench_q1_sf10_compact.json 2> $O/bench_q1_sf10_compact.err; echo "compact rc=$?"
TDP_FORCE_DIST=1 TDP_FORCE_COLLECTIVES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 200 --warmup 5 --no-cpu-baseline > $O/bench_q1_sf10_nccl_world1.json 2> $O/bench_q1_sf10_nccl_world1.err; echo "nccl rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_q1_reference_arm.json 2> $O/bench_q1_reference_arm.err; echo "ref rc=$?"
timeout 900 python bench.py --query q3 --steps 50 > $O/bench_q3_sf10.json 2> $O/bench_q3_sf10.err; echo "q3 rc=$?"
# SASS of the NVRTC-compiled fused scan (UBLKCP = bulk async copy, SYNCS = mbarrier)
mkdir -p $O/cubin
TDP_DUMP_CUBIN_DIR=$O/cubin timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-companion --e2e-steps 1 > /dev/null 2>&1
for f in $O/cubin/*.cubin; do cuobjdump -sass $f > ${f%.cubin}.sass 2>&1; done
grep -c "UBLKCP\|SYNCS" $O/cubin/*.sass
# ncu launch lists (cold-cache, serialised: share of the step, not absolute)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_q1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1 > /dev/null 2>&1; echo "ncu q1 rc=$?"
TDP_REPLAY=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_q3.csv python tools/profile_q3.py 10 > /dev/null 2>&1; echo "ncu q3 rc=$?"
ls -la $O

# ncu --set full of one compact-storage Q1 fused-scan launch (tdp_scan_agg).
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tdp_scan_agg --launch-skip 4 -c 1 -o gpurun_out/ncu/${1:-q1c} python bench.py --encoding compact ${2:-} --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-companion --e2e-steps 1 > gpurun_out/ncu/${1:-q1c}.log 2>&1; echo ncu rc=$?

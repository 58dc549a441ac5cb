mkdir -p gpurun_out
for cfg in "q1 wide" "q6 wide" "q1 compact" "q6 compact"; do set -- $cfg
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tdp_scan_agg -s 3 -c 1 --csv --log-file gpurun_out/traffic_$1_$2.csv python bench.py --query $1 --encoding $2 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-companion > /dev/null 2>&1; echo "$1 $2 rc=$?"; grep -E "dram__bytes|gpu__time" gpurun_out/traffic_$1_$2.csv | cut -d, -f10-20 | head -3
done

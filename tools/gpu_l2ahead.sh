# Q3 with the dense join's L2 bulk prefetch distance swept (TDP_L2_AHEAD)
mkdir -p gpurun_out
for a in 0 1 2 0.5; do
  TDP_L2_AHEAD=$a timeout 600 python bench.py --query q3 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/q3_a$a.json 2>gpurun_out/q3_a$a.err; echo "ahead $a rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/q3_a$a.json'));r=d['roofline'];print('ahead $a step',round(d['ms_per_step'],4),'eager',round(d['eager_ms_per_step'],4),'probe',round(r['kernel_ms'],4),r['frac'],d['parity']['status'])"
done
for a in 0 1; do
TDP_L2_AHEAD=$a TDP_REPLAY=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/l_q3_a$a.csv python tools/profile_q3.py 4 > /dev/null 2>&1; echo "ncu $a rc=$?"
python tools/launches.py gpurun_out/l_q3_a$a.csv 2>&1 | head -8
done

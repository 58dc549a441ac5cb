mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "llp or train or soft" > gpurun_out/pt_llp.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_llp.log
for g in 1 0; do
TDP_TRAIN_GRAPH=$g timeout 900 python bench.py --query llp --steps 10 --warmup 4 > gpurun_out/llp_g$g.json 2>gpurun_out/llp_g$g.err; echo "llp g=$g rc=$?"
python -c "import json;d=json.load(open('gpurun_out/llp_g$g.json'));r=d['roofline'];print('graph=$g step',round(d['value'],3),'frac',round(r['frac'],3),d['parity']['status'],d.get('graph'))"
done

mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for enc in wide compact; do for q in q1 q6; do
timeout 600 python bench.py --query $q --encoding $enc --steps 200 --no-cpu-baseline > gpurun_out/vb_${q}_$enc.json 2> gpurun_out/vb_${q}_$enc.err
python -c "
import json; d=json.load(open('gpurun_out/vb_${q}_$enc.json')); print('$q $enc', d['ms_per_step'], d['roofline']['frac'])"
done; done

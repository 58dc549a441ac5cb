mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "topk or order or limit or q3 or sort" 2>&1 | tail -3
timeout 300 python bench.py --query q3 --steps 20 --warmup 3 > gpurun_out/bench_q3.json 2> gpurun_out/bench_q3.err; python -c "
import json; d=json.load(open('gpurun_out/bench_q3.json')); print(d['ms_per_step'], d['eager_ms_per_step'], d['parity'])"
TDP_REPLAY=0 timeout 300 python tools/profile_q3.py 10 > gpurun_out/q3prof.txt 2>&1; head -30 gpurun_out/q3prof.txt

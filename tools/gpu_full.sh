mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 200 python tools/q3_eager.py
TDP_REPLAY=0 timeout 200 python tools/q3_eager.py

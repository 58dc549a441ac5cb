for kb in 200 216 224; do
TDP_RING_BUDGET_KB=$kb timeout 300 python bench.py --steps 300 --no-cpu-baseline --no-companion > gpurun_out/r_$kb.json 2>/dev/null; echo "q1 $kb $(grep -o '"ms_per_step.\{1,22\}\|kernel_ms.\{1,22\}' gpurun_out/r_$kb.json | tr '\n' ' ')"
TDP_RING_BUDGET_KB=$kb timeout 300 python bench.py --query q6 --steps 300 --no-cpu-baseline > gpurun_out/r6_$kb.json 2>/dev/null; echo "q6 $kb $(grep -o '"ms_per_step.\{1,22\}\|kernel_ms.\{1,22\}' gpurun_out/r6_$kb.json | tr '\n' ' ')"
done

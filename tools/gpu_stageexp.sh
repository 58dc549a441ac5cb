for ms in 4 3 2; do
TDP_RING_MIN_STAGES=$ms timeout 300 python bench.py --steps 300 --no-cpu-baseline --no-companion > gpurun_out/s_$ms.json 2>/dev/null; echo "q1 minstages=$ms $(grep -o '"ms_per_step.\{1,22\}\|kernel_ms.\{1,22\}' gpurun_out/s_$ms.json | tr '\n' ' ')"
TDP_RING_MIN_STAGES=$ms timeout 300 python bench.py --query q6 --steps 300 --no-cpu-baseline > gpurun_out/s6_$ms.json 2>/dev/null; echo "q6 minstages=$ms $(grep -o '"ms_per_step.\{1,22\}\|kernel_ms.\{1,22\}' gpurun_out/s6_$ms.json | tr '\n' ' ')"
done

for rb in 24 32 56; do
TDP_TWO_CTA_ROW_BYTES=$rb timeout 600 python bench.py --query q6 --steps 300 --no-cpu-baseline > gpurun_out/q6_$rb.json 2>/dev/null; echo "q6 rb=$rb $(grep -o '"ms_per_step.\{1,25\}\|kernel_ms.\{1,25\}' gpurun_out/q6_$rb.json | tr '\n' ' ')"
TDP_TWO_CTA_ROW_BYTES=$rb timeout 600 python bench.py --query q1 --steps 300 --no-cpu-baseline --no-companion > gpurun_out/q1_$rb.json 2>/dev/null; echo "q1 rb=$rb $(grep -o '"ms_per_step.\{1,25\}\|kernel_ms.\{1,25\}' gpurun_out/q1_$rb.json | tr '\n' ' ')"
done

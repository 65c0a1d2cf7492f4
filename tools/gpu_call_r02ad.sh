mkdir -p gpurun_out
for c in 2 1; do KS_REPS=3 KS_STEPS=20 timeout 300 python tools/knob_sweep.py $c '' 'D4ORM_K4CTA=4096' 'D4ORM_K4CTA=512'; done > gpurun_out/k4c2.log 2>&1

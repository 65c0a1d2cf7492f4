mkdir -p gpurun_out
for c in 2 3 4 1; do KS_REPS=3 KS_STEPS=20 timeout 300 python tools/knob_sweep.py $c '' 'D4ORM_K5REV=0'; done > gpurun_out/k5rev.log 2>&1

mkdir -p gpurun_out
for c in 2 3; do KS_REPS=3 KS_STEPS=20 timeout 300 python tools/knob_sweep.py $c '' 'D4ORM_K5CLASS=1' 'D4ORM_K5CLASS=1,D4ORM_K5REGEN=0' 'D4ORM_K5REGEN=1'; done > gpurun_out/k5class.log 2>&1

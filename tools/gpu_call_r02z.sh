mkdir -p gpurun_out
KS_REPS=3 KS_STEPS=20 timeout 300 python tools/knob_sweep.py 4 '' 'D4ORM_REGEN_SUB=4' 'D4ORM_REGEN_SUB=2' > gpurun_out/regensub.log 2>&1
for c in 2 3; do KS_REPS=3 KS_STEPS=20 timeout 300 python tools/knob_sweep.py $c 'D4ORM_K5CLASS=1,D4ORM_REGEN_SUB=4' 'D4ORM_K5CLASS=1,D4ORM_REGEN_SUB=2'; done >> gpurun_out/regensub.log 2>&1

mkdir -p gpurun_out
for i in 1 2 3; do KS_REPS=9 KS_STEPS=50 timeout 300 python tools/knob_sweep.py 1 '' 'D4ORM_FUSE_TAIL=0'; done > gpurun_out/tail_ab2.log 2>&1

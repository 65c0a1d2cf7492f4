mkdir -p gpurun_out
for c in 1 2 3 4; do KS_REPS=5 KS_STEPS=50 timeout 300 python tools/knob_sweep.py $c '' 'D4ORM_BENCH_ONEGRAPH=1' 'D4ORM_BENCH_ONEGRAPH=1,D4ORM_FUSE_TAIL=0' 'D4ORM_BENCH_ONEGRAPH=1,D4ORM_PDL=0'; done > gpurun_out/onegraph.log 2>&1

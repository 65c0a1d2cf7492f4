mkdir -p gpurun_out
for c in 1 2 5; do KS_REPS=3 KS_STEPS=20 timeout 300 python tools/knob_sweep.py $c '' 'D4ORM_BENCH_ONEGRAPH=0'; done > gpurun_out/onegraph2.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/t_suite_o.log 2>&1; echo "rc=$?" >> gpurun_out/t_suite_o.log
timeout 900 python bench.py > gpurun_out/bench_r02o.log 2>&1; echo "rc=$?" >> gpurun_out/bench_r02o.log

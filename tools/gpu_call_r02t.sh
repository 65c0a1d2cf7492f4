mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tail.py tests/test_gpu_parity.py tests/test_gpu_wfloor.py tests/test_gpu_checked.py -q > gpurun_out/t_k4c.log 2>&1; echo "rc=$?" >> gpurun_out/t_k4c.log
for c in 3 4; do KS_REPS=3 KS_STEPS=20 timeout 300 python tools/knob_sweep.py $c '' 'D4ORM_K4CLUSTER=0' '' 'D4ORM_K4CLUSTER=0'; done > gpurun_out/k4c.log 2>&1

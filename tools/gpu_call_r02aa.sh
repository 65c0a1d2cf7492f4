mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/t_sub4.log 2>&1; echo "rc=$?" >> gpurun_out/t_sub4.log
timeout 900 python -m pytest tests/test_gpu_e2e_f32.py -q -k "4" > gpurun_out/t_sub4_e2e.log 2>&1; echo "rc=$?" >> gpurun_out/t_sub4_e2e.log
KS_REPS=3 KS_STEPS=20 timeout 300 python tools/knob_sweep.py 4 '' > gpurun_out/sub4.log 2>&1

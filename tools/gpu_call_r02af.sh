mkdir -p gpurun_out
KS_BATCH=32768 KS_REPS=3 KS_STEPS=20 timeout 600 python tools/knob_sweep.py 5 '' 'D4ORM_K5REGEN=0' '' 'D4ORM_K5REGEN=0' > gpurun_out/regen8.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k run_graph > gpurun_out/t_rg.log 2>&1; echo "rc=$?" >> gpurun_out/t_rg.log

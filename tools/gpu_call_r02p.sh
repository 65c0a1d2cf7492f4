mkdir -p gpurun_out
for i in 1 2; do KS_REPS=5 KS_STEPS=50 timeout 300 python tools/knob_sweep.py 1 '' 'D4ORM_SEGS=8'; done > gpurun_out/segs.log 2>&1
timeout 600 python -m pytest tests/test_gpu_seg.py tests/test_gpu_tail.py tests/test_gpu_parity.py tests/test_gpu_checked.py -q > gpurun_out/t_segs.log 2>&1; echo "rc=$?" >> gpurun_out/t_segs.log

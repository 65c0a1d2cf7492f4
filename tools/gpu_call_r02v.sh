mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tail.py tests/test_gpu_checked.py tests/test_gpu_parity.py tests/test_gpu_baselines.py tests/test_gpu_regen.py -q > gpurun_out/t_tree.log 2>&1; echo "rc=$?" >> gpurun_out/t_tree.log
for c in 2 3 4 5; do KS_REPS=3 KS_STEPS=20 timeout 300 python tools/knob_sweep.py $c '' 'D4ORM_TREEPAR=0'; done > gpurun_out/tree_ab.log 2>&1

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tail.py -q > gpurun_out/t_tree.log 2>&1; echo "rc=$?" >> gpurun_out/t_tree.log

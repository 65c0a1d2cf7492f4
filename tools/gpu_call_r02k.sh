set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tail.py -q > gpurun_out/t_tail.log 2>&1; echo "rc=$?" >> gpurun_out/t_tail.log
timeout 300 python tools/knob_sweep.py 1 '' 'D4ORM_FUSE_TAIL=0' '' 'D4ORM_FUSE_TAIL=0' > gpurun_out/tail_ab.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/t_suite_k.log 2>&1; echo "rc=$?" >> gpurun_out/t_suite_k.log

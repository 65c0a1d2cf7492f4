set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_checked.py tests/test_reference_callers.py tests/test_dropin_cpp.py -m gpu -q > gpurun_out/t_f.log 2>&1; echo "rc=$?" >> gpurun_out/t_f.log
timeout 300 python tools/f64_c5.py 2 16384 > gpurun_out/f64.log 2>&1; echo "rc=$?" >> gpurun_out/f64.log
timeout 600 python tools/f64_c5.py 2 > gpurun_out/f64_full.log 2>&1; echo "rc=$?" >> gpurun_out/f64_full.log

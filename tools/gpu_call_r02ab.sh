mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/t_sub4.log 2>&1; echo "rc=$?" >> gpurun_out/t_sub4.log

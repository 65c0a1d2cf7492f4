mkdir -p gpurun_out
timeout 600 python tools/scaling_projection.py > gpurun_out/scaling_proj.log 2>&1; echo "rc=$?" >> gpurun_out/scaling_proj.log

mkdir -p gpurun_out
START=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/t_full_m24.log 2>&1; echo "rc=$? wall=$(( $(date +%s) - START ))s" >> gpurun_out/t_full_m24.log
timeout 900 python bench.py > gpurun_out/bench_m24.log 2>&1; echo "rc=$?" >> gpurun_out/bench_m24.log
timeout 600 python tools/step_profile.py 5 10 > gpurun_out/sp_m24.log 2>&1

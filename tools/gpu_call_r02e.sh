set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/t_suite_e.log 2>&1; echo "rc=$?" >> gpurun_out/t_suite_e.log
timeout 300 python tools/sanitize.py > gpurun_out/sanitize_plain.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_plain.log
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 50 python tools/sanitize.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rollout_fitness|k_wmean_regen|k_score_weights|k_wmean_tree" -s 8 -c 4 -o gpurun_out/c5_r02e -f python tools/ncu_k23.py 5 > gpurun_out/ncu_r02e.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_r02e.log
START=$(date +%s); timeout 2000 python -m pytest tests/test_gpu_e2e_f32.py -m gpu -q -s --durations=0 > gpurun_out/t_e2e.log 2>&1; echo "rc=$? wall=$(( $(date +%s) - START ))s" >> gpurun_out/t_e2e.log

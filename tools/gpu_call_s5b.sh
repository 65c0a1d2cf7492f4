set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/t_suite_s5b.log 2>&1; echo "rc=$?" >> gpurun_out/t_suite_s5b.log
tail -4 gpurun_out/t_suite_s5b.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rollout_fitness|k_wmean_regen|k_score_weights|k_wmean_tree" -s 8 -c 4 -o gpurun_out/c5_s5b -f python tools/ncu_k23.py 5 > gpurun_out/ncu_s5b.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_s5b.log
tail -3 gpurun_out/ncu_s5b.log

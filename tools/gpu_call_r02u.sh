mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rollout_fitness|k_wmean_regen|k_score_weights|k_wmean_tree" -s 8 -c 4 -o gpurun_out/c4_r02u -f python tools/ncu_k23.py 4 > gpurun_out/ncu_c4.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_c4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rollout_fitness|k_wmean|k_score_weights|k_small" -s 8 -c 4 -o gpurun_out/c2_r02u -f python tools/ncu_k23.py 2 > gpurun_out/ncu_c2.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_c2.log

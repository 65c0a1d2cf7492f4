mkdir -p gpurun_out
bash tools/round_bench.sh r02_s5c
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rollout_fitness|k_wmean_regen|k_score_weights|k_wmean_tree" -s 8 -c 4 -o gpurun_out/c5_s5i -f python tools/ncu_k23.py 5 > gpurun_out/ncu_s5i.log 2>&1; tail -2 gpurun_out/ncu_s5i.log

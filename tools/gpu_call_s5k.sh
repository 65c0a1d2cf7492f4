mkdir -p gpurun_out
bash tools/round_bench.sh r02_s5e
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rollout_fitness|k_wmean_regen|k_score_weights|k_wmean_tree" -s 8 -c 4 -o gpurun_out/c5_s5k -f python tools/ncu_k23.py 5 > gpurun_out/ncu_s5k.log 2>&1; tail -2 gpurun_out/ncu_s5k.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rollout_fitness" -s 2 -c 1 -o gpurun_out/c2_s5k -f python tools/ncu_k23.py 2 > gpurun_out/ncu_s5k2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rollout_fitness" -s 2 -c 1 -o gpurun_out/c4_s5k -f python tools/ncu_k23.py 4 > gpurun_out/ncu_s5k4.log 2>&1
python tools/scaling_projection.py | tee gpurun_out/scaling_projection_s5k.jsonl
timeout 900 python -m pytest tests -m "gpu and not slow" -q 2>&1 | tail -3

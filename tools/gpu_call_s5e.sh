mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_small.py -x -q 2>&1 | tail -5
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rollout_fitness" -s 2 -c 1 -o gpurun_out/c2_s5e -f python tools/ncu_k23.py 2 > gpurun_out/ncu_s5e.log 2>&1; tail -2 gpurun_out/ncu_s5e.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rollout_fitness" -s 2 -c 1 -o gpurun_out/c4_s5e -f python tools/ncu_k23.py 4 > gpurun_out/ncu_s5e4.log 2>&1; tail -2 gpurun_out/ncu_s5e4.log

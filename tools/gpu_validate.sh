# One GPU call that validates a build: full GPU suite, smoke, the round bench lines, an ncu --set full
# capture of a C5 step and the scaling projection (gpurun --timeout 4200 -- bash tools/gpu_validate.sh).
mkdir -p gpurun_out
START=$(date +%s)
timeout 3000 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/t_full_s5l.log 2>&1; echo "rc=$? wall=$(( $(date +%s) - START ))s" >> gpurun_out/t_full_s5l.log
tail -5 gpurun_out/t_full_s5l.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s5l.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_s5l.log; tail -2 gpurun_out/smoke_s5l.log
bash tools/round_bench.sh r02_s5f
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rollout_fitness|k_wmean_regen|k_score_weights|k_wmean_tree" -s 8 -c 4 -o gpurun_out/c5_s5l -f python tools/ncu_k23.py 5 > gpurun_out/ncu_s5l.log 2>&1; tail -2 gpurun_out/ncu_s5l.log
python tools/scaling_projection.py | tee gpurun_out/scaling_projection_s5l.jsonl

mkdir -p gpurun_out
START=$(date +%s)
timeout 3000 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/t_full_s5g.log 2>&1; echo "rc=$? wall=$(( $(date +%s) - START ))s" >> gpurun_out/t_full_s5g.log
tail -25 gpurun_out/t_full_s5g.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s5g.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_s5g.log; tail -3 gpurun_out/smoke_s5g.log

mkdir -p gpurun_out
START=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/t_full_q.log 2>&1; echo "rc=$? wall=$(( $(date +%s) - START ))s" >> gpurun_out/t_full_q.log
PYTHONPATH=. timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_q.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_q.log

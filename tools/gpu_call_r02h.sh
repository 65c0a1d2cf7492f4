set -x
mkdir -p gpurun_out
for c in 1 2 3 4 5; do timeout 300 python tools/knob_sweep.py $c '' 'D4ORM_PDL=0' '' 'D4ORM_PDL=0'; done > gpurun_out/pdl_ab.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/t_suite_h.log 2>&1; echo "rc=$?" >> gpurun_out/t_suite_h.log

set -x
mkdir -p gpurun_out
for c in 1 2 3 4 5; do timeout 300 python tools/exp_variants.py $c paper_2503_12204_b200/libd4orm_exp_pdl1.so paper_2503_12204_b200/libd4orm_b200.so paper_2503_12204_b200/libd4orm_exp_pdl1.so paper_2503_12204_b200/libd4orm_b200.so; done > gpurun_out/pdl_trig.log 2>&1
for c in 1 2 3 4; do timeout 300 python tools/knob_sweep.py $c '' ''; done >> gpurun_out/pdl_trig.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/t_suite_i.log 2>&1; echo "rc=$?" >> gpurun_out/t_suite_i.log
for c in 3 4; do timeout 300 python tools/knob_sweep.py $c '' 'D4ORM_K4CTA=16384' '' 'D4ORM_K4CTA=16384'; done > gpurun_out/k4cta.log 2>&1

set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_weighted_mean.py tests/test_gpu_multirank.py tests/test_reference_callers.py tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_dropin_cpp.py -m gpu -q -x > gpurun_out/t_new.log 2>&1; echo "rc=$?" >> gpurun_out/t_new.log
for c in 2 3 4; do timeout 300 python tools/exp_variants.py $c paper_2503_12204_b200/libd4orm_b200.so paper_2503_12204_b200/libd4orm_exp_minb4.so paper_2503_12204_b200/libd4orm_exp_minb6.so paper_2503_12204_b200/libd4orm_exp_minb7.so; done > gpurun_out/variants.log 2>&1
PYTHONPATH=.:tests timeout 1500 python tests/e2e_f32.py --configs 1,3 --sources philox --control --json gpurun_out/e2e_ctrl.json > gpurun_out/e2e_ctrl.log 2>&1; echo rc=$? >> gpurun_out/e2e_ctrl.log

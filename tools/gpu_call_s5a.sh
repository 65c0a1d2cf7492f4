set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pl32.py -x -q > gpurun_out/t_pl32.log 2>&1; echo "rc=$?" >> gpurun_out/t_pl32.log
tail -5 gpurun_out/t_pl32.log
timeout 300 python tools/knob_sweep.py 5 'D4ORM_PL32=0' '' > gpurun_out/pl32_ab.log 2>&1
timeout 600 python tools/exp_variants.py 5 paper_2503_12204_b200/libd4orm_exp_b5k8.so paper_2503_12204_b200/libd4orm_exp_b4k16.so paper_2503_12204_b200/libd4orm_exp_b5k4.so >> gpurun_out/pl32_ab.log 2>&1
cat gpurun_out/pl32_ab.log

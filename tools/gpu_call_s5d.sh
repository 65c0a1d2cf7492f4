mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_small.py -x -q 2>&1 | tail -15
for c in 2 3 4; do
  timeout 300 python tools/knob_sweep.py $c 'D4ORM_SMALL=0' '' 2>&1
  timeout 300 python tools/exp_variants.py $c paper_2503_12204_b200/libd4orm_exp_sm6.so paper_2503_12204_b200/libd4orm_exp_sm7k8.so 2>&1
done | tee gpurun_out/small_ab.log

set -x
mkdir -p gpurun_out
for c in 5 4; do timeout 300 python tools/exp_variants.py $c paper_2503_12204_b200/libd4orm_exp_base.so paper_2503_12204_b200/libd4orm_b200.so paper_2503_12204_b200/libd4orm_exp_base.so paper_2503_12204_b200/libd4orm_b200.so; done > gpurun_out/regen_ab.log 2>&1
timeout 300 python -m pytest tests/test_gpu_regen.py tests/test_gpu_wfloor.py -q > gpurun_out/t_regen.log 2>&1; echo "rc=$?" >> gpurun_out/t_regen.log
for c in 2 3 4; do timeout 400 python tools/knob_sweep.py $c '' 'D4ORM_SPC=4' 'D4ORM_SPC=16' 'D4ORM_TB=16' 'D4ORM_ZKEEP=0' 'D4ORM_CULL=0'; done > gpurun_out/knobs.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02g.log 2>&1; echo "rc=$?" >> gpurun_out/bench_r02g.log

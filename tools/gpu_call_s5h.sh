mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pl32.py -x -q 2>&1 | tail -3
timeout 300 python tools/knob_sweep.py 5 '' 2>&1 | tee gpurun_out/robotcull_ab.log
timeout 600 python tools/exp_variants.py 5 paper_2503_12204_b200/libd4orm_exp_rg1.so paper_2503_12204_b200/libd4orm_exp_rg5.so paper_2503_12204_b200/libd4orm_exp_rg6.so 2>&1 | tee -a gpurun_out/robotcull_ab.log
timeout 300 python tools/exp_phases.py 5 2>&1 | tee -a gpurun_out/robotcull_ab.log

mkdir -p gpurun_out
timeout 300 python tools/exp_variants.py 5 paper_2503_12204_b200/libd4orm_b200.so paper_2503_12204_b200/libd4orm_exp_plflat.so paper_2503_12204_b200/libd4orm_b200.so paper_2503_12204_b200/libd4orm_exp_plflat.so > gpurun_out/plflat.log 2>&1

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pl32.py -x -q 2>&1 | tail -3
D4ORM_LIB=$PWD/paper_2503_12204_b200/libd4orm_exp_split1.so timeout 900 python -m pytest tests/test_gpu_pl32.py -x -q 2>&1 | tail -3
timeout 600 python tools/exp_variants.py 5 paper_2503_12204_b200/libd4orm_exp_b5k8.so paper_2503_12204_b200/libd4orm_b200.so paper_2503_12204_b200/libd4orm_exp_split1.so paper_2503_12204_b200/libd4orm_b200.so 2>&1 | tee gpurun_out/pl32_ab2.log

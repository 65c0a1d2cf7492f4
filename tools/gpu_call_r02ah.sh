mkdir -p gpurun_out
for lib in libd4orm_b200 libd4orm_exp_m26 libd4orm_exp_m24; do D4ORM_LIB=$PWD/paper_2503_12204_b200/$lib.so timeout 600 python tools/step_profile.py 5 10 > gpurun_out/sp_$lib.log 2>&1; done

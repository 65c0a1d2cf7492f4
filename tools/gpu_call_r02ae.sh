mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r02ae.log 2>&1; echo "rc=$?" >> gpurun_out/bench_r02ae.log

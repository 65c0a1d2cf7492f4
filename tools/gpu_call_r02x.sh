mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r02x.log 2>&1; echo "rc=$?" >> gpurun_out/bench_r02x.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5_r02x.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-configs --no-f64 > gpurun_out/ncu_launch.log 2>&1

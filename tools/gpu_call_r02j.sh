set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r02j.log 2>&1; echo "rc=$?" >> gpurun_out/bench_r02j.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_r02j_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_r02j_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5_r02j.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-configs --no-f64 > gpurun_out/ncu_launch.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launch.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c1_r02j.csv python bench.py --config 1 --steps 10 --warmup 3 --no-cpu --no-e2e --no-f64 > gpurun_out/ncu_launch1.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launch1.log

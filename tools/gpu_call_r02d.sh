set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_reference_callers.py tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_dropin_cpp.py tests/test_gpu_fullsize.py -m gpu -q > gpurun_out/t_new2.log 2>&1; echo "rc=$?" >> gpurun_out/t_new2.log
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02d.log 2>&1; echo "rc=$?" >> gpurun_out/bench_r02d.log
PYTHONPATH=.:tests timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02d.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_r02d.log
/usr/bin/time -v timeout 1800 python -m pytest tests/test_gpu_e2e_f32.py -m gpu -q -s --durations=0 > gpurun_out/t_e2e.log 2>&1; echo "rc=$?" >> gpurun_out/t_e2e.log

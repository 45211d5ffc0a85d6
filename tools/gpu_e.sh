set -x
python -m pytest tests/test_gpu_parity.py tests/test_trajectories_gpu.py tests/test_full_size_gpu.py -m gpu -q -rf --timeout 1200 -p no:cacheprovider > gpurun_out/r02e_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02e_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-beyond-l2 > gpurun_out/r02e_bench.log 2>&1
echo "bench rc $?"; tail -c 1500 gpurun_out/r02e_bench.log

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -rf --timeout 1200 -p no:cacheprovider > gpurun_out/r02a_pytest.log 2>&1
echo "pytest rc $?"
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/r02a_bench.log 2>&1
echo "bench rc $?"
tail -3 gpurun_out/r02a_pytest.log

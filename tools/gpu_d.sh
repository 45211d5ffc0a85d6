set -x
bash tools/reference_suite.sh run
python -m pytest tests -m gpu -q -rf --timeout 1200 -p no:cacheprovider > gpurun_out/r02d_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02d_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02d_bench.log 2>&1
echo "bench rc $?"; tail -c 3000 gpurun_out/r02d_bench.log

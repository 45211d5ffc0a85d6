set -x
python -m pytest tests/test_design_graph_gpu.py -m gpu -q -rf -x --timeout 900 -p no:cacheprovider > gpurun_out/r02g_pytest.log 2>&1
echo "pytest rc $?"; tail -30 gpurun_out/r02g_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-beyond-l2 > gpurun_out/r02g_bench.log 2>&1
echo "bench rc $?"; tail -c 800 gpurun_out/r02g_bench.log

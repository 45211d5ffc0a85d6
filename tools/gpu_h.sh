python -m pytest tests/test_design_graph_gpu.py tests/test_gpu_parity.py tests/test_trajectories_gpu.py -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/r02h_pytest.log 2>&1
echo "pytest rc $?"; grep -E "^E  |passed|failed" gpurun_out/r02h_pytest.log | head -30

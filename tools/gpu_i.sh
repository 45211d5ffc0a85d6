python -m pytest tests -m gpu -q -rf --timeout 1200 -p no:cacheprovider > gpurun_out/r02i_pytest.log 2>&1
echo "pytest rc $?"; grep -E "^E  |passed|failed|^FAILED" gpurun_out/r02i_pytest.log | head -30

python -m pytest tests/test_slab_gpu.py tests/test_slab_nccl_gpu.py -m gpu -q -rfs --timeout 900 -p no:cacheprovider > gpurun_out/r02k_pytest.log 2>&1
echo "pytest rc $?"; grep -E "^E  |passed|failed|^FAILED|SKIP" gpurun_out/r02k_pytest.log | head -20
timeout 900 python bench.py --mode slab --config c4 --iters 5 --steps 3 --warmup 1 > gpurun_out/r02k_slab_c4.log 2>&1
echo "slab rc $?"; tail -c 1500 gpurun_out/r02k_slab_c4.log

python -m pytest tests/test_gpu_parity.py tests/test_full_size_gpu.py tests/test_preconditioner_gpu.py tests/test_slab_gpu.py -m gpu -q -rf --timeout 1200 -p no:cacheprovider > gpurun_out/r02r_pytest.log 2>&1
echo "pytest rc $?"; grep -E "^E  |passed|failed|^FAILED" gpurun_out/r02r_pytest.log | head -20
for L in 1 0; do OTM_K10_LOCK=$L timeout 900 python bench.py --config c4 --iters 20 --steps 2 --warmup 1 --no-cpu --no-c1 --no-beyond-l2 > gpurun_out/r02r_c4_lock$L.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r02r_c4_lock$L.log').read().strip().splitlines()[-1]); print('lock $L', d['value'], d['roofline']['achieved'], d['roofline']['frac'], {k:(round(v['ms'],1), v['gbs'] and round(v['gbs'])) for k,v in d['kernels'].items()})"; done
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-c1 > gpurun_out/r02r_c3.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/r02r_c3.log').read().strip().splitlines()[-1]); print('c3', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline_beyond_l2']['frac'], {k:(round(v['ms'],1), v['gbs'] and round(v['gbs'])) for k,v in d['kernels'].items()})"

python -m pytest tests/test_slab_gpu.py -m gpu -q -rfs --timeout 900 -p no:cacheprovider > gpurun_out/r02l_pytest.log 2>&1
echo "pytest rc $?"; grep -E "^E  |passed|failed|^FAILED" gpurun_out/r02l_pytest.log | head -20
timeout 900 python bench.py --mode slab --config c4 --iters 5 --steps 3 --warmup 1 > gpurun_out/r02l_slab_c4.log 2>&1
echo "slab rc $?"; python -c "
import json; d=json.loads(open('gpurun_out/r02l_slab_c4.log').read().strip().splitlines()[-1]); print(d['value'], d['single_gpu'], d['slab_over_single'])"
OTM_SLAB_GRAPH=0 timeout 900 python bench.py --mode slab --config c4 --iters 5 --steps 3 --warmup 1 --no-single > gpurun_out/r02l_slab_c4_nograph.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/r02l_slab_c4_nograph.log').read().strip().splitlines()[-1]); print('nograph', d['value'])"
for b in 1 2; do OTM_OC_BPS=$b timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-beyond-l2 --no-c1 > gpurun_out/r02l_oc_bps$b.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r02l_oc_bps$b.log').read().strip().splitlines()[-1]); print('bps $b', d['value'], d['kernels']['oc'])"; done

python -m pytest tests -m gpu -q -rfs --timeout 1200 -p no:cacheprovider > gpurun_out/r02p_pytest.log 2>&1
echo "pytest rc $?"; grep -E "^E  |passed|failed|^FAILED" gpurun_out/r02p_pytest.log | head -20
python tools/slab_diag2.py c4
timeout 900 python bench.py --mode slab --config c4 --iters 5 --steps 3 --warmup 1 > gpurun_out/r02p_slab_c4.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/r02p_slab_c4.log').read().strip().splitlines()[-1]); print(d['value'], d['single_gpu']['value'], d['slab_over_single'])"

python -m pytest tests/test_preconditioner_gpu.py tests/test_design_graph_gpu.py -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/r02j_pytest.log 2>&1
echo "pytest rc $?"; grep -E "^E  |passed|failed|^FAILED" gpurun_out/r02j_pytest.log | head -20
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-beyond-l2 > gpurun_out/r02j_bench.log 2>&1
echo "bench rc $?"; python -c "
import json; d=json.loads(open('gpurun_out/r02j_bench.log').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['c3_to_convergence']['value'], {k:(round(v['ms'],1)) for k,v in d['kernels'].items()}, d['solver_stats'])"
OTM_TILE=0 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-beyond-l2 --no-c1 > gpurun_out/r02j_bench_notile.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/r02j_bench_notile.log').read().strip().splitlines()[-1]); print('notile', d['value'], d['e2e']['value'], {k:(round(v['ms'],1)) for k,v in d['kernels'].items()})"

# level-0 stencil GB/s (bench kernel classes) for each env setting
for v in "$@"; do
  env $v timeout 300 python bench.py --iters 100 --steps 1 --warmup 3 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); k=d['kernels']; print('$v', round(d['value'],4), 'l0', round(k['l0_stencil']['gbs']), round(k['l0_stencil']['ms']/k['l0_stencil']['launches']*1e3,1), 'us/launch', 'vcycle', round(k['vcycle']['ms'],1))"
done

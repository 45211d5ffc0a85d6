# res64 class time per launch for env settings
for v in "$@"; do
  env $v timeout 300 python bench.py --iters 100 --steps 1 --warmup 3 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); k=d['kernels']; print('$v', round(d['value'],4), 'res64', round(k['res64']['ms']/k['res64']['launches']*1e3,1), 'us/launch', round(k['res64']['gbs']), 'GB/s; restrict/vcycle', round(k['vcycle']['ms'],1))"
done

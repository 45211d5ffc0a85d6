# usage: bash tools/cmp_env.sh "ENV=1 ..." "X=0" ...   (A/B timing of env knobs, 200-iteration c3 structures)
# TESTENV="ENV=..." runs the GPU tests under that environment first
env $TESTENV timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -1
for v in "$@"; do
  env $v timeout 300 python bench.py --iters 200 --steps 2 --warmup 3 --no-cpu --no-prof 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['value'],4), d['e2e']['value'])"
done

#!/bin/bash
# A/B of env knobs on 200-iteration c3 structures with solver statistics:
#   bash tools/knob.sh "OTM_TOLF=0.5" "OTM_TOLF=0.8" ...
for v in "$@"; do
  env $v OTM_STATS=1 timeout 300 python bench.py --iters 200 --steps 2 --warmup 3 --no-cpu --no-prof > /tmp/k.out 2> /tmp/k.err
  python -c "import sys,json; d=json.loads(open('/tmp/k.out').readlines()[-1]); print('$v', round(d['value'],4), round(d['e2e']['value'],4))"
  grep "stats" /tmp/k.err | tail -1
done

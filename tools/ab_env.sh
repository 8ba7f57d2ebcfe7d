#!/bin/bash
# A/B of one environment switch on the C4 bench (experiments only): tools/ab_env.sh VAR v1 v2 ...
var=$1; shift
for e in "$@" "$@"; do
  env $var=$e timeout 600 python bench.py --steps 10 --warmup 3 --fc-steps 2 --no-e2e --no-cpu-baseline > gpurun_out/ab_$e.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_$e.json')); print('$var=$e', round(d['ms_per_step'],3), d['kernel_ms_per_iter'], 'fc', round(d['fc']['ms_per_iter'],3))"
done

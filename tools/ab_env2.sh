#!/bin/bash
# A/B of environment settings on the C4 IC bench (experiments): tools/ab_env2.sh "A=1 B=2" "A=0" ...
for i in 1 2; do
for e in "$@"; do
  env $e timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-fc --no-c2 > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$e', round(d['ms_per_step'],4), d['kernel_ms_per_iter'])"
done
done

#!/bin/bash
# FC / e2e A/B of library variants (lib/variants/NAME.so; "main" = default build), experiments only
for i in 1 2; do
for v in "$@"; do
  if [ $v = main ]; then L=""; else L="PBA_GPU_LIB=$PWD/paper_1704_06967_b200/lib/variants/$v.so"; fi
  env $L timeout 400 python bench.py --steps 10 --warmup 3 --fc-steps 3 --no-cpu-baseline --no-c2 > gpurun_out/abfc.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/abfc.json')); print('$v', 'ic', round(d['ms_per_step'],4), 'fc', round(d['fc']['ms_per_iter'],3), d['fc']['kernel_ms'], 'e2e', round(d['e2e']['ms_per_step'],2))" 2>/dev/null || echo "$v failed"
done
done

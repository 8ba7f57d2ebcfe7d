#!/bin/bash
# A/B of library variants (lib/variants/NAME.so; "main" = the default build) on the C4 IC bench (experiments)
for i in 1 2; do
for v in "$@"; do
  if [ $v = main ]; then L=""; else L="PBA_GPU_LIB=$PWD/paper_1704_06967_b200/lib/variants/$v.so"; fi
  env $L timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-fc --no-c2 > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$v', round(d['ms_per_step'],4), d['kernel_ms_per_iter'])" 2>/dev/null || echo "$v failed"
done
done

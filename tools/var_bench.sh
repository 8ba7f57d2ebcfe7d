#!/bin/bash
# A/B timing of library variants (experiments only): IC iteration on C4, no FC/e2e/cpu legs.
for v in "$@"; do
  PBA_GPU_LIB=$PWD/paper_1704_06967_b200/lib/variants/$v.so timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-fc --no-e2e --no-cpu-baseline > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python -c "import json; d=json.load(open('gpurun_out/var_$v.json')); print('$v', round(d['ms_per_step'],3), 'obs', round(d['roofline']['launch_ms'],3), 'frac', round(d['roofline']['frac'],3), d['kernel_ms_per_iter'])"
done

#!/bin/bash
# A/B timing of library variants on the FC leg (experiments only): C4, FC iterations.
for v in "$@"; do
  PBA_GPU_LIB=$PWD/paper_1704_06967_b200/lib/variants/$v.so timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --fc-steps 3 --no-e2e --no-cpu-baseline > gpurun_out/varfc_$v.json 2> gpurun_out/varfc_$v.err
  python -c "import json; d=json.load(open('gpurun_out/varfc_$v.json')); f=d['fc']; print('$v', round(f['ms_per_iter'],3), f['kernel_ms'], 'ic', round(d['ms_per_step'],3))" || tail -3 gpurun_out/varfc_$v.err
done

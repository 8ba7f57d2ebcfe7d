#!/bin/bash
# A/B timing of library variants (experiments only): IC + FC iteration and IC build on C4.
for v in "$@"; do
  PBA_GPU_LIB=$PWD/paper_1704_06967_b200/lib/variants/$v.so timeout 600 python bench.py --config C4 --steps 5 --warmup 2 --fc-steps 2 --no-e2e --no-cpu-baseline > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python -c "import json; d=json.load(open('gpurun_out/var_$v.json')); print('$v', 'IC', round(d['ms_per_step'],3), 'obs', round(d['roofline']['launch_ms'],3), 'FC', round(d['fc']['ms_per_iter'],2), d['fc']['kernel_ms'], 'build+1st', d['setup_s']['ic_build_and_first_pass'])"
done

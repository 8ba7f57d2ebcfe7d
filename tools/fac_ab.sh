timeout 600 python -m pytest -q -x tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_failures.py 2>&1 | tail -3
for e in "PBA_CHOL_INV=0" "PBA_CHOL_INV=1"; do
  env $e timeout 400 python bench.py --steps 10 --warmup 3 --fc-steps 3 --no-cpu-baseline --no-c2 > gpurun_out/fac.json 2>gpurun_out/fac.err
  python -c "import json; d=json.load(open('gpurun_out/fac.json')); print('$e', 'ic', round(d['ms_per_step'],4), d['kernel_ms_per_iter'], 'fc', round(d['fc']['ms_per_iter'],3), d['fc']['kernel_ms'], 'e2e', round(d['e2e']['ms_per_step'],2))" || tail -5 gpurun_out/fac.err
done

set -u
for i in 1 2; do
for v in main v1; do
  if [ $v = main ]; then L=""; else L="PBA_GPU_LIB=$PWD/paper_1704_06967_b200/lib/variants/$v.so"; fi
  env $L timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-fc --no-c2 > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', round(d['ms_per_step'],4), d['kernel_ms_per_iter'])"
done
done
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_full_size.py tests/test_gpu_edges.py 2>&1 | tail -3

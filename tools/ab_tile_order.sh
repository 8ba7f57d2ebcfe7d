for e in 0 1 0 1; do
  PBA_TILE_ORDER=$e timeout 600 python bench.py --steps 10 --warmup 3 --fc-steps 2 --no-e2e --no-cpu-baseline > gpurun_out/to_$e.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/to_$e.json')); print('order=$e', round(d['ms_per_step'],3), d['kernel_ms_per_iter'], 'fc', round(d['fc']['ms_per_iter'],3), d['fc']['kernel_ms']['obs_pass'])"
done

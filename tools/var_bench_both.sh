for v in ${VARIANTS:-base rx base rx}; do
  PBA_GPU_LIB=$PWD/paper_1704_06967_b200/lib/variants/$v.so timeout 600 python bench.py --steps 10 --warmup 3 --fc-steps 3 --no-e2e --no-cpu-baseline --no-c2 > gpurun_out/v_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/v_$v.json')); print('$v', round(d['ms_per_step'],3), d['kernel_ms_per_iter']['obs_pass'], 'fc', round(d['fc']['ms_per_iter'],3), d['fc']['kernel_ms']['obs_pass'])"
done

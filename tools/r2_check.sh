#!/bin/bash
# Round-2 change check on one B200: focused GPU tests, then the C4 bench line (IC, FC, e2e, C2).
timeout 1200 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_sharding.py tests/test_golden.py \
  tests/test_gpu_failures.py tests/test_multihost.py 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2_check.json 2> gpurun_out/r2_check.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2_check.json"))
print("ic", round(d["ms_per_step"], 4), d["kernel_ms_per_iter"])
print("fc", round(d["fc"]["ms_per_iter"], 3), d["fc"]["kernel_ms"])
print("e2e", round(d["e2e"]["ms_per_step"], 2), d["e2e"]["step_ms"])
print("c2", round(d["c2_joint"]["ms_per_iter"], 3))
PY

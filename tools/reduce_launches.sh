#!/bin/bash
# ncu launch list of the point-major / tile reduction kernels for library variants (experiments only).
for v in "$@"; do
  PBA_GPU_LIB=$PWD/paper_1704_06967_b200/lib/variants/$v.so timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"k_backsub|k_point|k_cf|k_finalize|k_gauge" --csv --log-file gpurun_out/red_$v.csv \
    python tools/profile_obs.py --config C4 --iters 3 > gpurun_out/red_$v.log 2>&1
  python - "$v" <<'PY'
import csv, sys, collections
v = sys.argv[1]
rows = [r for r in csv.DictReader(l for l in open(f"gpurun_out/red_{v}.csv") if not l.startswith("==")) if r.get("Metric Name") == "gpu__time_duration.sum"]
agg = collections.defaultdict(list)
for r in rows:
    agg[r["Kernel Name"].split("(")[0][-40:]].append(float(r["Metric Value"]) / (1e3 if r["Metric Unit"] == "usecond" else 1e6 if r["Metric Unit"] == "nsecond" else 1))
print(v, {k: (len(x), round(sum(x) / len(x), 4)) for k, x in agg.items()})
PY
done

"""Merge the BASELINE C5 sweep (tools/c5_run.sh): the timing / oracle rows of gpurun_out/r2_c5_sweep.jsonl
with the per-size ncu metric captures gpurun_out/r2_c5_ncu_<N>_<k>.csv of the IC pass, into one JSON line
per size (profiles/r2_c5_sweep.jsonl).  The ncu figures are per launch (average over the captured
launches of k_obs_lane_tab): DRAM bytes, DRAM GB/s and its fraction of the measured peak, FP64-pipe,
issue and occupancy percentages, L2 hit rate.

  python tools/c5_merge.py [gpurun_out] > profiles/r2_c5_sweep.jsonl"""
import csv
import json
import sys
from pathlib import Path

src = Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out")
SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def ncu_row(path, peak_gbs):
    if not path.exists() or path.stat().st_size == 0:
        return None
    rows = list(csv.DictReader(open(path)))
    per = {}
    for r in rows:
        per.setdefault(r["ID"], {})[r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
    if not per:
        return None
    n = len(per)

    def avg(name, conv=lambda v, u: v):
        vals = [conv(*m[name]) for m in per.values() if name in m]
        return sum(vals) / len(vals) if vals else None

    ms = avg("gpu__time_duration.sum", lambda v, u: v * SCALE.get(u, 1e-6))
    rd = avg("dram__bytes_read.sum", lambda v, u: v * BYTES.get(u, 1.0))
    wr = avg("dram__bytes_write.sum", lambda v, u: v * BYTES.get(u, 1.0))
    gbs = (rd + wr) / (ms / 1e3) / 1e9
    return {"launches": n, "pass_ms": round(ms, 4), "dram_bytes": rd + wr, "dram_GBs": round(gbs, 1),
            "dram_frac": round(gbs / peak_gbs, 3),
            "fp64_pipe_pct": round(avg("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"), 1),
            "issue_active_pct": round(avg("smsp__issue_active.avg.pct_of_peak_sustained_active"), 1),
            "warps_active_pct": round(avg("sm__warps_active.avg.pct_of_peak_sustained_active"), 1),
            "l2_hit_pct": round(avg("lts__t_sector_hit_rate.pct"), 1),
            "note": "IC passes of one handle, per launch (ncu --clock-control none, cold caches, serialised launches)"}


for line in open(src / "r2_c5_sweep.jsonl"):
    line = line.strip()
    if not line.startswith("{"):
        continue
    row = json.loads(line)
    row["ncu"] = ncu_row(src / f"r2_c5_ncu_{row['points']}_{row['k_target']}.csv", row.get("peak_GBs") or 6547.8)
    print(json.dumps(row))

"""Summarise ncu outputs for profiles/: per-kernel launch shares from a
gpu__time_duration launch list, and key counters from a --set full report."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__grid_size", "sm__cycles_elapsed.avg.per_second",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                 "second": 1e3, "s": 1e3}
        ms = v * scale.get(unit, 1e-6)
        name = r["Kernel Name"].split("(")[0]
        per[name][0] += 1
        per[name][1] += ms
    # the library's kernels (anonymous namespace k_*); torch's scene-generation kernels are reported
    # as one aggregate line
    ours = {k: v for k, v in per.items() if "unnamed>::k_" in k}
    other = [sum(v[0] for k, v in per.items() if k not in ours), sum(v[1] for k, v in per.items() if k not in ours)]
    tot = sum(v[1] for v in ours.values())
    out = {k: {"launches": v[0], "total_ms": round(v[1], 4), "share": round(v[1] / tot, 4)}
           for k, v in sorted(ours.items(), key=lambda kv: -kv[1][1])}
    out["(not this library: torch scene generation, excluded from the shares)"] = {
        "launches": other[0], "total_ms": round(other[1], 4), "share": None}
    return out


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:80]}
        for i, k in enumerate(hdr):  # the listed counters plus every FP64 / DMMA / tensor-pipe counter
            if k in KEYS or any(t in k for t in ("dmma", "pipe_fp64", "pipe_tensor", "fp64")):
                if vals[i] not in ("", "n/a"):
                    d[k] = f"{vals[i]} {units[i]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if kind == "launches" else full(path), indent=1))

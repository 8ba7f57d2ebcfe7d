#!/bin/bash
# Compact ncu metric set for one kernel of library variants (experiments only).
# usage: tools/ncu_metrics.sh KERNEL_REGEX variant...
K=$1; shift
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_global_op_ld.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active,l1tex__m_xbar2l1tex_read_bytes.sum
for v in "$@"; do
  PBA_GPU_LIB=$PWD/paper_1704_06967_b200/lib/variants/$v.so timeout 600 ncu --metrics $M --clock-control none --kernel-name-base mangled -k regex:"$K" --launch-skip 1 -c 1 --csv python tools/profile_obs.py --config C4 --iters 2 2>/dev/null | grep -v "^==" > gpurun_out/met_$v.csv
  python - "$v" <<'PY'
import csv, sys
v = sys.argv[1]
rows = list(csv.DictReader(open(f"gpurun_out/met_{v}.csv")))
print(v, rows[0]["Kernel Name"][:40] if rows else "none")
for r in rows: print("   ", r["Metric Name"], r["Metric Value"], r["Metric Unit"])
PY
done

#!/bin/bash
# BASELINE C5 grid on one B200: timing + oracle checks, then an ncu metric capture of the IC pass per size.
out=gpurun_out
timeout 3000 python tools/c5_sweep.py > $out/r2_c5_sweep.jsonl 2> $out/r2_c5_sweep.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct
for n in 250000 500000 1000000 2000000 4000000; do for k in 8 16 32 64; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:k_obs_lane_tab --launch-skip 0 -c 2 --csv \
    python tools/c5_sweep.py --profile $n:$k 2>/dev/null | grep -v "^==" > $out/r2_c5_ncu_${n}_${k}.csv
done; done

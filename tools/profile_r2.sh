#!/bin/bash
# Round-2 measurement on one B200: the default bench line, the ncu launch list of a short bench run,
# and one `ncu --set full` capture of each hot kernel (IC pass, FC pass, IC build, SYRK, dataflow
# factorization, reduce kernels).  Outputs under gpurun_out/ (summaries go to profiles/).
set -u
out=gpurun_out
timeout 600 python bench.py > $out/p2_bench.json 2> $out/p2_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file $out/p2_launches.csv \
  python bench.py --steps 2 --warmup 3 --fc-steps 2 --no-cpu-baseline --no-c2 > $out/p2_ncu_launch.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none --kernel-name-base function \
  -k regex:"k_obs_lane|k_point|k_cf|k_backsub|k_schur_syrk|k_chol_tiles|k_bdot" -c 16 \
  -o $out/p2_full -f python tools/profile_obs.py --config C4 --iters 2 --fc > $out/p2_ncu_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function \
  -k regex:"k_obs_lane" -c 4 -o $out/p2_full_ic -f python tools/profile_obs.py --config C4 --iters 3 > $out/p2_ncu_full_ic.log 2>&1
ls -la $out/p2_*

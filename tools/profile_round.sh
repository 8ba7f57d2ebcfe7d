#!/bin/bash
# Round-end measurement on one B200 (run under gpurun from the repo root):
#   GPU tests, the default bench line, the ncu launch list of a short bench run and one
#   `ncu --set full` capture of each hot kernel.  Outputs under gpurun_out/ (copy the
#   summaries into profiles/ with tools/ncu_summary.py).
set -u
out=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $out/p_tests.log 2>&1; echo "tests rc=$?" >> $out/p_tests.log
timeout 600 python bench.py > $out/p_bench.json 2> $out/p_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file $out/p_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $out/p_ncu_launch.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base function \
  -k regex:"k_obs_lane|k_point|k_cf|k_backsub|k_schur_syrk|k_chol_inv" -c 14 \
  -o $out/p_full -f python tools/profile_obs.py --config C4 --iters 3 > $out/p_ncu_full.log 2>&1
tail -2 $out/p_tests.log

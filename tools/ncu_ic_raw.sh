#!/bin/bash
# One `ncu --set full` capture of the IC pass at C4 (plus the pipe/L1 breakdown metrics) and its raw CSV page.
set -u
out=gpurun_out
lib=${PBA_GPU_LIB:-}
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function \
  --metrics sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_cbu.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_active,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_global_op_ld.sum,sm__mio_inst_issued.avg.pct_of_peak_sustained_active,idc__requests.sum,idc__request_cycles_active.avg.pct_of_peak_sustained_active,sm__mio2rf_writeback_active.avg.pct_of_peak_sustained_active \
  -k regex:"k_obs_lane_tab" -s 1 -c 1 -o $out/${1:-icraw} -f python tools/profile_obs.py --config C4 --iters 3 > $out/${1:-icraw}.log 2>&1
ncu -i $out/${1:-icraw}.ncu-rep --page raw --csv > $out/${1:-icraw}_raw.csv 2>/dev/null
ncu -i $out/${1:-icraw}.ncu-rep --page details --csv > $out/${1:-icraw}_details.csv 2>/dev/null
ls -la $out/${1:-icraw}*

#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers
for wl in ${WLS:-cfg4_k64_f64 cfg4_k128_f64}; do
  PROF_WL=$wl timeout 900 ncu --metrics $M --clock-control none -k 'regex:^(?!at::|void at::).*' --csv \
    python scripts/profile_suite.py > gpurun_out/r02_ncu_$wl.csv 2> gpurun_out/r02_ncu_$wl.err
done

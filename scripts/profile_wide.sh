#!/bin/bash
# ncu metric capture of the wide FP64 tensor-core kernels at config 4 (k=128, B=64, n=32768).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size,smsp__issue_active.avg.pct_of_peak_sustained_active
for k in ${KS:-64 128}; do
  ncu --metrics $M --clock-control none -k regex:'k_(chol_mw|chol_dmma|subset_mw|vchol_dmma|vsub_dmma)$' --csv \
    python scripts/time_wide_vjp.py $k > gpurun_out/wide_ncu_vjp_$k.csv 2> gpurun_out/wide_ncu_vjp_$k.err
  ncu --metrics $M --clock-control none -k regex:'k_(chol_mw|chol_dmma|subset_mw|vchol_dmma|vsub_dmma)$' --csv \
    python scripts/time_wide_fwd.py $k > gpurun_out/wide_ncu_fwd_$k.csv 2> gpurun_out/wide_ncu_fwd_$k.err
done

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SWEEP_WL=cfg4_k64_f64 SWEEP_PEROP=1 SWEEP_ENV=";BGM_VSUB_WARPS=8;BGM_WIDE_DMMA_WARPS=2;BGM_SUBSET_WARPS=2;BGM_SUBSET_WARPS=1;BGM_WIDE_BURN=256;BGM_WIDE_BURN=320" timeout 1200 python scripts/sweep_suite.py > gpurun_out/r2l_k64.jsonl 2> gpurun_out/r2l_k64.err
SWEEP_WL=cfg4_k128_f64 SWEEP_PEROP=1 SWEEP_ENV=";BGM_VSUB_WARPS=4;BGM_WIDE_DMMA_WARPS=8;BGM_WIDE_DMMA_WARPS=2;BGM_SUBSET_WARPS=4;BGM_WIDE_BURN=512;BGM_WIDE_BURN=640" timeout 1500 python scripts/sweep_suite.py > gpurun_out/r2l_k128.jsonl 2> gpurun_out/r2l_k128.err

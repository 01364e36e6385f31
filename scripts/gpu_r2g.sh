#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SWEEP_WL=cfg3 SWEEP_B=256,128,64,32 SWEEP_ENV="BGM_T1_WARPS=2.5;BGM_T1_WARPS=3;BGM_T1_WARPS=3.5;BGM_T1_WARPS=4;BGM_T1_WARPS=5;BGM_T1_WARPS=6" timeout 900 python scripts/sweep_suite.py > gpurun_out/r2g_cfg3.jsonl 2> gpurun_out/r2g_cfg3.err
SWEEP_WL=cfg1 SWEEP_B=4096,512 SWEEP_PEROP=1 SWEEP_ENV=";BGM_NARROW_SEGF=2;BGM_NARROW_SEGF=1;BGM_NARROW_SEGF=1,BGM_NARROW_BURN=24;BGM_NARROW_SEGF=2,BGM_NARROW_BURN=48;BGM_NARROW_SEGF=1,BGM_NARROW_BURN=48" timeout 900 python scripts/sweep_suite.py > gpurun_out/r2g_cfg1.jsonl 2> gpurun_out/r2g_cfg1.err
SWEEP_WL=cfg4_k64_f64 SWEEP_B=64,8 SWEEP_PEROP=1 SWEEP_ENV="" timeout 900 python scripts/sweep_suite.py > gpurun_out/r2g_cfg4.jsonl 2> gpurun_out/r2g_cfg4.err

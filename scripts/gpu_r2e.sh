#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_mlik_gpu.py -x -q > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2e_pytest.log
SWEEP_B=32,64,256 SWEEP_BURN=96,64,48,32 SWEEP_SEG=0,48,64,96,128,192 SWEEP_TILE=32,1 timeout 1200 python scripts/sweep_small_b.py > gpurun_out/r2e_sweep.jsonl 2> gpurun_out/r2e_sweep.err

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
./oracle/_ref/scaling_dropin > gpurun_out/r2k_scaling_dropin.json 2>&1
./oracle/_ref/scaling_ref > gpurun_out/r2k_scaling_ref.json 2>&1
python scripts/time_dropin_ops.py > gpurun_out/r2k_dropin_ops.log 2>&1

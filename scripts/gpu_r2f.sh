#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for b in 96 64 48; do
BGM_BURN=$b BGM_DEBUG=1 timeout 300 python scripts/debug_burn.py > gpurun_out/r2f_burn$b.log 2>&1
done

#!/bin/bash
# A/B of library variants: $@ = list of .so paths (in-tree default first)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
WL=${AB_WL:-cfg3}; BS=${AB_B:-256,32}
for rep in 1 2; do
for lib in paper_1902_10078_b200/libbandgm_b200.so "$@"; do
  BGM_LIBRARY=$PWD/$lib SWEEP_WL=$WL SWEEP_B=$BS timeout 600 python scripts/sweep_suite.py 2>&1 | sed "s|^|$lib |"
done
done

#!/bin/bash
# Round profile capture: launch list of one bench run + full captures of the
# two config-3 sweeps.  Outputs under gpurun_out/ (copied to profiles/ by hand).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_bench_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e \
  > gpurun_out/${TAG}_ncu_launches.log 2>&1
for k in k_fwd k_bwd; do
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:^${k}\$" -s 1 -c 1 \
    -o gpurun_out/${TAG}_$k python scripts/profile_mlik.py > gpurun_out/${TAG}_ncu_$k.log 2>&1
done
ls -la gpurun_out | tail

#!/bin/bash
# Round-2 profile capture: launch list of one default bench run, full ncu
# captures of the config-3 sweeps, and of config 4's top kernels.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-proxy > gpurun_out/${TAG}_bench_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-proxy \
  > gpurun_out/${TAG}_ncu_launches.log 2>&1
for k in k_fwd k_bwd; do
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:^${k}\$" -s 1 -c 1 \
    -o gpurun_out/${TAG}_$k python scripts/profile_mlik.py > gpurun_out/${TAG}_ncu_$k.log 2>&1
done
ls -la gpurun_out | tail

#!/bin/bash
# A/B: the suite's independent operators on concurrent stream lanes (with and
# without a high-priority critical lane) vs serial
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for w in cfg4_k64_f64 cfg4_k128_f64 cfg4_k64_f32; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-proxy > gpurun_out/lanesP_$w.json 2> gpurun_out/lanesP_$w.err
  BENCH_LANE_PRIO=0 timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-proxy > gpurun_out/lanes0_$w.json 2> gpurun_out/lanes0_$w.err
done

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for w in cfg3 cfg1 cfg2 cfg4_k64_f64 cfg4_k64_f32 cfg4_k128_f64 cfg4_k128_f32; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r2j_bench_$w.json 2> gpurun_out/r2j_bench_$w.err
done
for w in cfg3 cfg1 cfg2 cfg4_k64_f64; do
  timeout 900 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > gpurun_out/r2j_ref_$w.json 2> gpurun_out/r2j_ref_$w.err
done
./oracle/_ref/scaling_dropin > gpurun_out/r2j_scaling_dropin.json 2>&1
./oracle/_ref/scaling_ref > gpurun_out/r2j_scaling_ref.json 2>&1

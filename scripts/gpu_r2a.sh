#!/bin/bash
# round-2 first GPU pass: new fused-step test, bench lines for every workload
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mlik_gpu.py -x -q > gpurun_out/r2a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
for w in cfg3 cfg1 cfg2 cfg4_k64_f64 cfg4_k64_f32 cfg4_k128_f64 cfg4_k128_f32; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/r2a_bench_$w.json 2> gpurun_out/r2a_bench_$w.err
  echo "$w rc=$?" >> gpurun_out/r2a_status.log
done

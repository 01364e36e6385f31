#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_mlik_gpu.py -x -q > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2d_pytest.log
timeout 600 python scripts/debug_proxy.py 256 128 64 32 33 8 > gpurun_out/r2d_proxy.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_proxy.log
for w in cfg3 cfg1 cfg4_k64_f64; do
timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/r2d_bench_$w.json 2> gpurun_out/r2d_bench_$w.err
done

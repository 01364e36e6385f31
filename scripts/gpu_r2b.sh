#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_mlik_gpu.py -x -q > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
CUDA_LAUNCH_BLOCKING=1 timeout 600 python scripts/debug_proxy.py 256 128 64 32 > gpurun_out/r2b_proxy.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_proxy.log
timeout 600 python bench.py --workload cfg1 --steps 10 --warmup 3 --no-proxy > gpurun_out/r2b_bench_cfg1.json 2> gpurun_out/r2b_bench_cfg1.err

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_mlik_gpu.py -x -q > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c_pytest.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python scripts/debug_proxy.py 128 > gpurun_out/r2c_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_memcheck.log

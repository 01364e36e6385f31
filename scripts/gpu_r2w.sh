#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_wide_gpu.py tests/test_configs_gpu.py tests/test_promote_gpu.py -q -x > gpurun_out/r2w_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_pytest.log
AB_WL=cfg4_k64_f64 AB_B=64 SWEEP_PEROP=1 bash scripts/gpu_ab.sh build_var/libold.so
AB_WL=cfg4_k128_f64 AB_B=64 SWEEP_PEROP=1 bash scripts/gpu_ab.sh build_var/libold.so

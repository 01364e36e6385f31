#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_wide_gpu.py tests/test_configs_gpu.py -q -x -k "wide or cfg4 or config4 or chol" > gpurun_out/r2n_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_pytest.log
AB_WL=cfg4_k128_f64 AB_B=64,8 bash scripts/gpu_ab.sh build_var/libold.so

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_narrow_gpu.py tests/test_kernels_gpu.py tests/test_configs_gpu.py tests/test_promote_gpu.py tests/test_dropin.py -q -x > gpurun_out/r2x_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2x_pytest.log
AB_WL=cfg1 AB_B=4096,512 SWEEP_PEROP=1 bash scripts/gpu_ab.sh build_var/libold.so

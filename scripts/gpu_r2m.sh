#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mlik_gpu.py tests/test_configs_gpu.py -q -x -k "mlik or config3 or cfg3" > gpurun_out/r2m_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_pytest.log
AB_WL=cfg3 AB_B=256,32 bash scripts/gpu_ab.sh build_var/libb0.so

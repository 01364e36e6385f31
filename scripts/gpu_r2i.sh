#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_promote_gpu.py tests/test_dropin.py tests/test_autograd_gpu.py -q > gpurun_out/r2i_new.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_new.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2i_all.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_all.log

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mlik_gpu.py tests/test_narrow_gpu.py -x -q > gpurun_out/r2h_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2h_pytest.log
SWEEP_WL=cfg3 SWEEP_B=256,128,32 SWEEP_ENV=";BGM_T1_WARPS_F=3;BGM_T1_WARPS_B=3;BGM_T1_WARPS_B=5;BGM_T1_WARPS_F=5;BGM_T1_WARPS_F=3,BGM_T1_WARPS_B=3;BGM_T1_WARPS=2" timeout 900 python scripts/sweep_suite.py > gpurun_out/r2h_cfg3.jsonl 2> gpurun_out/r2h_cfg3.err
timeout 900 python bench.py --workload cfg1 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2h_bench_cfg1.json 2> gpurun_out/r2h_bench_cfg1.err
timeout 900 python bench.py --workload cfg3 --steps 20 --warmup 5 > gpurun_out/r2h_bench_cfg3.json 2> gpurun_out/r2h_bench_cfg3.err

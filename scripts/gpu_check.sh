#!/bin/bash
# One GPU session: tests, smoke, bench.  Logs under gpurun_out/.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
echo "== pytest gpu" ; timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
for wl in ${BENCH_WORKLOADS:-cfg3}; do
  echo "== bench $wl"; timeout ${BENCH_TIMEOUT:-900} python bench.py --workload $wl --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_$wl.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench_$wl.log
done

#!/bin/bash
# Round-end evidence in one GPU session: GPU tests, smoke, the bench (both
# arms), the launch list of the bench command, per-op suites of configs 1-4.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r01}
bash scripts/gpu_check.sh
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; echo "reference rc=$?"; tail -1 gpurun_out/bench_reference.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1; echo "ncu rc=$?"
python scripts/launch_summary.py gpurun_out/${TAG}_launches.csv "ncu --metrics gpu__time_duration.sum --clock-control none -c 400 $CMD" \
  > gpurun_out/${TAG}_launch_summary.txt
timeout 1200 python scripts/bench_ops.py --configs 1,2,3,4 > gpurun_out/${TAG}_ops.jsonl 2> gpurun_out/${TAG}_ops.err; echo "ops rc=$?"
grep -h suite_frac gpurun_out/${TAG}_ops.jsonl | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l); print(d['config'], d['dtype'], d['suite_ms'], d['suite_roofline_ms'], d['suite_frac'])"

#!/bin/bash
# config-4 warp-count knobs, one process each (they are read once per process)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() {  # tag workload env...
  local tag=$1 w=$2; shift 2
  env "$@" timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-proxy > gpurun_out/knob_${tag}_$w.json 2> gpurun_out/knob_${tag}_$w.err
}
for w in cfg4_k64_f64 cfg4_k128_f64; do
  run base $w X=1
  run vsub8 $w BGM_VSUB_WARPS=8
  run vsub4 $w BGM_VSUB_WARPS=4
  run sub2 $w BGM_SUBSET_WARPS=2
  run sub8 $w BGM_SUBSET_WARPS=8
  run chol2 $w BGM_WIDE_DMMA_WARPS=2
  run chol8 $w BGM_WIDE_DMMA_WARPS=8
done

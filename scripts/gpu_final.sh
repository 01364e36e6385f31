#!/bin/bash
# Evidence refresh: full GPU suite, every bench workload, config-3 ncu captures.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r2f}
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gputests.log
for w in cfg3 cfg1 cfg2 cfg4_k64_f64 cfg4_k64_f32 cfg4_k128_f64 cfg4_k128_f32; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err
done
TAG=r02 bash scripts/profile_r02.sh > gpurun_out/${T}_profile.log 2>&1
for k in k_fwd k_bwd; do
  ncu -i gpurun_out/r02_$k.ncu-rep --page raw --csv > gpurun_out/r02_${k}_raw.csv 2>/dev/null
  ncu -i gpurun_out/r02_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_${k}_sass.csv 2>/dev/null
  rm -f gpurun_out/r02_$k.ncu-rep
done

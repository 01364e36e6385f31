#!/bin/bash
# Evidence refresh: full GPU suite, smoke, every bench workload (both arms for
# the headline), config-3 ncu captures reduced to CSV.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r2f}
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gputests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
SECONDS=0; timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench_cfg3.json 2> gpurun_out/${T}_bench_cfg3.err
echo "bench wall ${SECONDS}s" > gpurun_out/${T}_bench_cfg3.time; SECONDS=0; timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_ref_cfg3.json 2> gpurun_out/${T}_ref_cfg3.err
echo "ref wall ${SECONDS}s" > gpurun_out/${T}_ref_cfg3.time
for w in cfg1 cfg2 cfg4_k64_f64 cfg4_k64_f32 cfg4_k128_f64 cfg4_k128_f32; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err
done
for w in cfg1 cfg2 cfg4_k64_f64 cfg4_k128_f64; do
  timeout 900 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > gpurun_out/${T}_ref_$w.json 2> gpurun_out/${T}_ref_$w.err
done

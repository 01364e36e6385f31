#!/bin/bash
# A/B of library builds on the config-3 bench: scripts/ab_bench.sh LIB_A LIB_B [rounds]
cd "$(dirname "$0")/.." || exit 1
for r in $(seq ${3:-3}); do
  for lib in "$1" "$2"; do
    BGM_LIBRARY=$lib python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1]); k = d['roofline']['kernel_ms']
print('$lib'.split('/')[-2], d['ms_per_step'], 'fwd', k['mlik_t1_fwd'], 'bwd', k['mlik_t1_bwd'])"
  done
done

#!/bin/bash
# Config-1 burn-in / segment-length sweep (solve_vec, cholesky) via the
# narrow kernels' environment overrides; one line per setting.
cd "$(dirname "$0")/.." || exit 1
for burn in ${BURNS:-default 32 48 64}; do
  for segf in ${SEGFS:-1 2 3 4 6}; do
    env $([ $burn != default ] && echo BGM_NARROW_BURN=$burn) BGM_NARROW_SEGF=$segf timeout 120 \
      python scripts/bench_ops.py --configs ${CFG:-1} 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print('burn $burn segf $segf', d['suite_ms'], ' '.join(f\"{o['op']}={o['ms']}\" for o in d['ops']))"
  done
done

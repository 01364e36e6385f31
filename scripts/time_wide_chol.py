"""Wide Cholesky alone at config-4 size (fp64): median of 7 event-timed calls per
bandwidth, max |L - L_ref| against the BGM_REF_WARPS build-in variant when asked.
python scripts/time_wide_chol.py [k ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import factor

for k in [int(a) for a in sys.argv[1:]] or (64, 128):
    dev = torch.device("cuda", 0)
    B, n = 64, 32768
    L0 = factor(B, n, k, torch.float64, dev, 0.02 / k ** 0.5, 105, tile=1)
    Q = bgm.product_band_band_restricted(L0, bgm.T(L0), k, 0)
    L = bgm.cholesky(Q)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        bgm.cholesky(Q, check=False)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    err = (L.data - L0.data).abs().max().item()
    print(f"k={k} cholesky {sorted(ts)[3]:.3f} ms  (min {min(ts):.3f})  max|L - L0| {err:.3e}  env {os.environ.get('BGM_WIDE_DMMA_WARPS', '-')}", flush=True)

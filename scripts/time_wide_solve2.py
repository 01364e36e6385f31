"""Wide solves alone at config-4 size: median of 7 event-timed calls per bandwidth and direction;
max |x - x_ref| against float64 numpy-free residual check: |L x - v| / |v|.
python scripts/time_wide_solve2.py [k ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import factor

for k in [int(a) for a in sys.argv[1:]] or (64, 128):
    dev = torch.device("cuda", 0)
    B, n = 64, 32768
    L = factor(B, n, k, torch.float64, dev, 0.02 / k ** 0.5, 105, tile=1)
    v = bgm.Vecs(torch.randn(B, n, dtype=torch.float64, device=dev), B, n, 1)
    for tr in (False, True):
        x = bgm.solve_vec(L, v, transpose_l=tr)
        torch.cuda.synchronize()
        back = bgm.product_band_vec(L, x, transpose_b=tr)
        res = ((back.data - v.data).abs().max() / v.data.abs().max()).item()
        ts = []
        for _ in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            bgm.solve_vec(L, v, transpose_l=tr, check=False)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"k={k} solve {'Lt' if tr else 'L '} {sorted(ts)[3]:.3f} ms (min {min(ts):.3f})  residual {res:.2e}  "
              f"blk={os.environ.get('BGM_WSOLVE_BLK', '1')} units={os.environ.get('BGM_WSOLVE_UNITS', '-')}", flush=True)

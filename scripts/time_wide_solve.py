"""Wide solve_vec (L and L^T) at config-4 size, fp64, reference layout."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import factor, normal_vec, timeit

dev = torch.device("cuda", 0)
for k in [int(a) for a in sys.argv[1:]] or (64, 128):
    B, n = 64, 32768
    L0 = factor(B, n, k, torch.float64, dev, 0.02 / k ** 0.5, 105, tile=1)
    Q = bgm.product_band_band_restricted(L0, bgm.T(L0), k, 0)
    L = bgm.cholesky(Q)
    b = normal_vec(B, n, torch.float64, dev, 42, tile=1)
    t0 = timeit(lambda: bgm.solve_vec(L, b, False, check=False), 3)
    t1 = timeit(lambda: bgm.solve_vec(L, b, True, check=False), 3)
    print(f"k={k} solve L {t0:.3f} ms  L^T {t1:.3f} ms", flush=True)

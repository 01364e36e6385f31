"""Narrow vjp_cholesky at config-3 size (B=256, n=65536, k=16, tile 32) and smaller k."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import factor, normal_band, timeit

dev = torch.device("cuda", 0)
for k in [int(a) for a in sys.argv[1:]] or (16, 8, 4):
    B, n = 256, 65536
    L = factor(B, n, k, torch.float64, dev, 0.1, 31)
    Q = bgm.product_band_band_restricted(L, bgm.T(L), k, 0)
    Lp = bgm.cholesky(Q)
    Lb = normal_band(B, n, k, 0, torch.float64, dev, 33)
    ms = timeit(lambda: bgm.vjp_cholesky(Lp, Lb), 5)
    print(f"k={k} vjp_cholesky {ms:.3f} ms", flush=True)

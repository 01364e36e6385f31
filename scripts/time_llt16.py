"""band(L L^T) lower at config 3 (B=256, n=65536, k=16, tile 32)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import factor, timeit

dev = torch.device("cuda", 0)
L = factor(256, 65536, 16, torch.float64, dev, 0.1, 31)
for _ in range(3):
    print("L.Lt lower ms", round(timeit(lambda: bgm.product_band_band_restricted(L, bgm.T(L), 16, 0), 5), 3), flush=True)

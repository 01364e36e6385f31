"""Times vjp_product_band_band at config-2 shapes (A (8,8), B (3,3)), B=512 n=65536."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import normal_band, timeit

dev = torch.device("cuda", 0)
B, n = 512, 65536
A = normal_band(B, n, 8, 8, torch.float64, dev, 22)
Bm = normal_band(B, n, 3, 3, torch.float64, dev, 23)
P2 = normal_band(B, n, 11, 11, torch.float64, dev, 26)
print(os.environ.get("BGM_STREAM_VAB", "0"), "vjp A.B ms", timeit(lambda: bgm.vjp_product_band_band(A, Bm, P2), 5))

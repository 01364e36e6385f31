"""A(8,8) B(3,3) product at config 2 (B=512, n=65536, tile 32)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import normal_band, timeit

dev = torch.device("cuda", 0)
A = normal_band(512, 65536, 8, 8, torch.float64, dev, 22)
Bm = normal_band(512, 65536, 3, 3, torch.float64, dev, 23)
print(os.environ.get("BGM_STREAM_VAR", "0"), "A.B ms", round(timeit(lambda: bgm.product_band_band(A, Bm), 5), 3))

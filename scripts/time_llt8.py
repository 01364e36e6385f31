"""L L^T full (8,8) at config 2 (B=512, n=65536, tile 32)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import normal_band, timeit

dev = torch.device("cuda", 0)
L = normal_band(512, 65536, 8, 0, torch.float64, dev, 21)
print(os.environ.get("BGM_STREAM_VAR", "0"), "L.Lt ms", round(timeit(lambda: bgm.product_band_band(L, bgm.T(L)), 5), 3))

"""vjp_log_det_from_cholesky at config-4 size (B=64, n=32768, k=64/128, tile 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import factor, timeit

dev = torch.device("cuda", 0)
for k in (64, 128):
    L = factor(64, 32768, k, torch.float64, dev, 0.02 / k ** 0.5, 41 + k, tile=1)
    print(k, "vjp_log_det ms", timeit(lambda: bgm.vjp_log_det_from_cholesky(L, 1.0), 5), flush=True)

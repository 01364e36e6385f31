"""vjp_solve_vec at config-4 (tile 1) and config-3 (tile 32) sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import factor, normal_vec, timeit

dev = torch.device("cuda", 0)
for (B, n, k, t) in ((64, 32768, 64, 1), (64, 32768, 128, 1), (256, 65536, 16, 32)):
    L = factor(B, n, k, torch.float64, dev, 0.02 / k ** 0.5, 41 + k, tile=t)
    x = normal_vec(B, n, torch.float64, dev, 3, tile=t)
    sb = normal_vec(B, n, torch.float64, dev, 4, tile=t)
    o = bgm.outer_band(x, sb, k, 0)
    print(k, t, "vjp_solve", round(timeit(lambda: bgm.vjp_solve_vec(L, x, sb, False, check=False), 5), 3),
          "outer", round(timeit(lambda: bgm.outer_band(x, sb, k, 0), 5), 3), flush=True)

"""Narrow solve_vec timings at config-3 (k=16) and config-1 (k=4) sizes, tile 32."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import factor, normal_vec, timeit

dev = torch.device("cuda", 0)
out = []
for (B, n, k) in ((256, 65536, 16), (4096, 2048, 4)):
    L0 = factor(B, n, k, torch.float64, dev, 0.1, 31)
    L = bgm.cholesky(bgm.product_band_band_restricted(L0, bgm.T(L0), k, 0))
    y = normal_vec(B, n, torch.float64, dev, 32)
    t0 = timeit(lambda: bgm.solve_vec(L, y, False, check=False), 5)
    t1 = timeit(lambda: bgm.solve_vec(L, y, True, check=False), 5)
    out.append(f"k={k}: L {t0:.3f} Lt {t1:.3f}")
print(os.environ.get("BGM_LIBRARY", "main").split("/")[-2] if "BGM_LIBRARY" in os.environ else "main", " | ".join(out))

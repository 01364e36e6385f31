"""Fast narrow solves vs the generic reference-loop kernel at config-3 size."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import factor, normal_vec

B, n, k = [(256, 65536, 16), (4096, 2048, 4)][int(sys.argv[1]) if len(sys.argv) > 1 else 0]
dev = torch.device("cuda", 0)
L0 = factor(B, n, k, torch.float64, dev, 0.1, 31)
Q = bgm.product_band_band_restricted(L0, bgm.T(L0), k, 0)
L = bgm.cholesky(Q)
y = normal_vec(B, n, torch.float64, dev, 32)
lib = bgm.library()
for tr in (False, True):
    a = bgm.solve_vec(L, y, tr).data
    lib.bgm_force_generic(1)
    r = bgm.solve_vec(L, y, tr).data
    lib.bgm_force_generic(0)
    err = ((a - r).abs() / r.abs().clamp_min(1e-300)).max().item()
    print("transpose", tr, "max rel err vs generic", err, "max |x|", r.abs().max().item())

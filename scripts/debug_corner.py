"""Does the fused config-3 step read input corner cells?  (It must not.)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1902_10078_b200 as bgm
from tests import common as cm

rng = np.random.default_rng(4)
for tile in (1, 32):
    for (B, n, k) in ((2, 40, 2), (2, 600, 16), (3, 700, 4)):
        L0 = cm.config_factor(rng, B, n, k)
        y = rng.normal(0, 1, (B, n))
        base = bgm.marginal_likelihood_grad(bgm.Bands.from_reference(L0, k, 0, tile=tile),
                                            bgm.Vecs.from_reference(y, tile=tile), 0.05)[0].cpu().numpy()
        P = L0.copy()
        for r in range(1, k + 1):
            P[:, n - r:, r] = 1e3  # corner cells of the last columns
        pert = bgm.marginal_likelihood_grad(bgm.Bands.from_reference(P, k, 0, tile=tile),
                                            bgm.Vecs.from_reference(y, tile=tile), 0.05)[0].cpu().numpy()
        print(f"tile={tile} B={B} n={n} k={k} loss change from poisoned corners: {np.abs(pert - base).max():.3e}")

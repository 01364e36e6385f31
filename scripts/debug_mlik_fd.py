"""Finite differences of the fused config-3 loss vs its L-bar / tau2-bar."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1902_10078_b200 as bgm
from tests import common as cm

rng = np.random.default_rng(4)
B, n, k, tau2 = 2, 40, 2, 0.05
L0 = cm.config_factor(rng, B, n, k)
y = rng.normal(0, 1, (B, n))
yd = bgm.Vecs.from_reference(y, tile=1)


def run(Lr, t=tau2):
    loss, lb, tb = bgm.marginal_likelihood_grad(bgm.Bands.from_reference(Lr, k, 0, tile=1), yd, t)
    return loss.cpu().numpy(), lb.numpy(), tb.cpu().numpy()


loss, lb, tb = run(L0)
h = 1e-6
worst = 0
for (b, j, r) in [(0, 0, 0), (0, 5, 1), (0, 17, 2), (1, 3, 0), (1, 30, 1), (0, 38, 1), (0, 39, 0)]:
    P, M = L0.copy(), L0.copy()
    P[b, j, r] += h
    M[b, j, r] -= h
    fd = (run(P)[0][b] - run(M)[0][b]) / (2 * h)
    print(f"cell b={b} j={j} r={r}: fd {fd:+.10f}  l_bar {lb[b, j, r]:+.10f}")
fdt = (run(L0, tau2 + h)[0] - run(L0, tau2 - h)[0]) / (2 * h)
print("tau2: fd", fdt, "tbar", tb)

"""Runs the config-2 band products and their VJPs once each (for ncu captures).
PROF_B matrices (default 128) of n = 65536, tile 32."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import normal_band, normal_vec

B = int(os.environ.get("PROF_B", "128"))
n = int(os.environ.get("PROF_N", "65536"))
dev = torch.device("cuda", 0)
L = normal_band(B, n, 8, 0, torch.float64, dev, 21)
Lt = L.transpose()
A = normal_band(B, n, 8, 8, torch.float64, dev, 22)
Bm = normal_band(B, n, 3, 3, torch.float64, dev, 23)
v = normal_vec(B, n, torch.float64, dev, 24)
P1 = normal_band(B, n, 8, 8, torch.float64, dev, 25)
P2 = normal_band(B, n, 11, 11, torch.float64, dev, 26)
pv = normal_vec(B, n, torch.float64, dev, 27)
for _ in range(int(os.environ.get("PROF_REPS", "1"))):
    bgm.product_band_band(L, bgm.T(L))
    bgm.product_band_band(A, Bm)
    bgm.product_band_vec(A, v)
    bgm.vjp_product_band_band(L, Lt, P1)
    bgm.vjp_product_band_band(A, Bm, P2)
    bgm.vjp_product_band_vec(A, v, pv, False)
torch.cuda.synchronize()
print("ok")
if os.environ.get("PROF_DL", "1") == "1":  # config-3 shapes: band(L L^T) lower and the dL VJP at k = 16
    del A, Bm, P1, P2
    L16 = normal_band(B, n, 16, 0, torch.float64, dev, 31)
    G16 = normal_band(B, n, 16, 0, torch.float64, dev, 34)
    L16t = L16.transpose()
    bgm.product_band_band_restricted(L16, bgm.T(L16), 16, 0)
    bgm.vjp_product_band_band(L16, L16t, G16)
    torch.cuda.synchronize()
    print("ok dl")
